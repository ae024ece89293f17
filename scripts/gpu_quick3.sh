cd $GRAFT_REPO_ROOT
for zb in "2 2" "2 4"; do set -- $zb
SOG_ZPASS=$1 SOG_ZPASS_B=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_z.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_z.log').read().strip().splitlines()[-1]);print('zpass $1 B $2', d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items() if 'mid' in k})" || tail -5 gpurun_out/bench_z.log
done
