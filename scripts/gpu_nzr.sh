#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -x -q -m gpu -k "c1_comp or c2_tol or shapes or edge or loopback or fp32 or confined" > gpurun_out/n_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/n_tests.log
for z in 1 2 3; do for c in c5 c4 c3 "c2 --tol 1e-8"; do
SOG_NEAR_NZR=$z timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bnz.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bnz.log').read().strip().splitlines()[-1]);print('nzr $z $c', '%.3f ms'%d['ms_per_step'], 'near %.2f'%d['stages_ms']['near'])" || tail -3 gpurun_out/bnz.log
done; done
