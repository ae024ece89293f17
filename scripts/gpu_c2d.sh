#!/bin/bash
for v in "--config c2 --tol 1e-8 --long-method direct" "--config c2 --tol 1e-12 --long-method direct" "--config t4 --window kb --long-method direct" "--config c2 --tol 1e-4 --long-method direct" "--config t2 --long-method direct"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $v > gpurun_out/bd.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bd.log').read().strip().splitlines()[-1]);print('$v', '%.3f ms'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items() if 'long' in k})" || tail -3 gpurun_out/bd.log
done
