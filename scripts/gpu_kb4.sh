#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kb.py tests/test_gpu_parity.py -x -q -m gpu -k "c1 or c2_tol or shapes or fp32 or edge or determinism" > gpurun_out/kb_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/kb_tests.log
for w in gs kb; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --window $w > gpurun_out/bench_$w.log 2>&1; echo bench_$w=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_$w.log').read().strip().splitlines()[-1]);print('$w', d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
done
for rc in 2.75 3.0 3.5; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --window kb --rc-factor $rc > gpurun_out/sw.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);p=d['config']['plan']
print('kb rc $rc', round(d['ms_per_step'],2), {k:p[k] for k in ('m','Ix','Izs','P','Ilx','Pc')}, {k:round(v,1) for k,v in d['stages_ms'].items() if v>0.5})" 2>&1 | tail -1
done
