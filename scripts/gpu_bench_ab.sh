# c5 bench A/B only (no tests): ms per step and selected stages for each env variant in $VARIANTS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:--}; do
  e=$(echo "$v" | tr "," " "); [ "$v" = "-" ] && e=""
  env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BARGS} > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/ab.log
done
