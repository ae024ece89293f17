#!/bin/bash
# quick: parity subset + c5 bench (window $1, default gs)
mkdir -p gpurun_out
w=${1:-gs}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py -x -q -m gpu -k "c1 or c2_tol or shapes or edge or fp32" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --window $w > gpurun_out/bench_q.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]);print('$w', d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
