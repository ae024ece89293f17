#!/bin/bash
# KB window: GPU parity tests + c5 bench (gs vs kb) + launch list of the kb run
mkdir -p gpurun_out
python -c "import paper_2412_04595_b200 as p; p.load_library()" > gpurun_out/build.log 2>&1; echo load=$?
timeout 1500 python -m pytest tests/test_gpu_kb.py tests/test_dist_gpu.py -x -q -m gpu > gpurun_out/kb_tests.log 2>&1; echo kbtests=$?; tail -15 gpurun_out/kb_tests.log
for w in gs kb; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --window $w > gpurun_out/bench_$w.log 2>&1; echo bench_$w=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_$w.log').read().strip().splitlines()[-1]);print('$w', d['ms_per_step'], d['config']['plan'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
done
