#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py -x -q -m gpu -k "shapes or c2_tol or confined or c1_stages or full_size_c2 or full_size_c3" > gpurun_out/tg_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/tg_tests.log
for v in "--config c3" "--config c2 --tol 1e-8" "--config c2 --tol 1e-12" "--config s1" "--config t4 --window kb" "--config c2 --tol 1e-4"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $v > gpurun_out/btg.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/btg.log').read().strip().splitlines()[-1]);print('$v', '%.3f ms'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items() if 'long' in k})" || tail -3 gpurun_out/btg.log
done
