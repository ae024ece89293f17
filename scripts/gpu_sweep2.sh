for rc in 2.75 3.0 3.25 3.5 3.75; do for eta in 0.3; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --eta $eta --rc-factor $rc > gpurun_out/sw.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);p=d['config']['plan']
print('rc $rc eta $eta', round(d['ms_per_step'],2), {k:p[k] for k in ('m','Ix','Izs','P','Ilx','Pc')}, {k:round(v,1) for k,v in d['stages_ms'].items() if v>0.5})" 2>&1 | tail -1
done; done
