#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_direct.py -x -q -m gpu > gpurun_out/direct_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/direct_tests.log
for cfg in c5 c4; do for lm in fft direct; do
timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --long-method $lm > gpurun_out/bench_${cfg}_$lm.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_${cfg}_$lm.log').read().strip().splitlines()[-1]);print('$cfg $lm', d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/bench_${cfg}_$lm.log
done; done
