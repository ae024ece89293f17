#!/bin/bash
mkdir -p gpurun_out
for v in "--config c5" "--config c4" "--config c3" "--config s1" "--config c2 --tol 1e-12" "--config c2 --tol 1e-8"; do for o in "" "--optimize"; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $v $o > gpurun_out/bo.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bo.log').read().strip().splitlines()[-1]);p=d['config']['plan'];print('$v $o', '%.3f ms'%d['ms_per_step'], 'rc %.2f m %d Ix %d Izs %d Pc %d'%(p['rc'],p['m'],p['Ix'],p['Izs'],p['Pc']))" || tail -3 gpurun_out/bo.log
done; done
