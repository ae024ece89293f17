#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "graph or c1_comp or determinism" > gpurun_out/g_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/g_tests.log
for v in "--config c2 --tol 1e-4" "--config c2 --tol 1e-8" "--config c4" "--config c5"; do for g in "" "--no-graph"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $v $g > gpurun_out/bg.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bg.log').read().strip().splitlines()[-1]);print('$v $g', '%.3f ms'%d['ms_per_step'], 'e2e %.3f ms'%d['e2e']['ms_per_step'])" || tail -3 gpurun_out/bg.log
done; done
