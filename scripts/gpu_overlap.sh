#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c1_comp or graph or determinism or c2_tol" > gpurun_out/o_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/o_tests.log
for m in off low high; do for c in c5 c4 "c2 --tol 1e-8"; do
SOG_NEAR_STREAM=$m timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bov.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bov.log').read().strip().splitlines()[-1]);print('$m $c', '%.3f ms'%d['ms_per_step'], 'e2e %.3f'%d['e2e']['ms_per_step'])" || tail -3 gpurun_out/bov.log
done; done
