#!/bin/bash
# build here, then run a command on the GPU box only if the build succeeded
cd /root/repo
python -c "import paper_2412_04595_b200.build as b; b.build()" > /tmp/build.log 2>&1 || { grep -v "ptxas warning" /tmp/build.log | tail -20; exit 1; }
timeout ${GPU_TIMEOUT:-1800} /usr/local/graft/bin/gpurun --timeout ${GPU_LIMIT:-900} -- "$@"
