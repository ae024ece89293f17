#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py tests/test_dist_gpu.py -x -q -m gpu -k "confined or shapes or c2_tol or c1 or loopback" > gpurun_out/s1_tests.log 2>&1; echo tests=$?; tail -4 gpurun_out/s1_tests.log
for w in gs kb; do
timeout 600 python bench.py --config s1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --window $w > gpurun_out/bench_s1_$w.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_s1_$w.log').read().strip().splitlines()[-1]);print('$w', d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/bench_s1_$w.log
done
