# parity (mid-path files) + c5 A/B for the env variants in $VARIANTS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py tests/test_dist_gpu.py ${EXTRA_TESTS} -q -x 2>&1 | tail -3
for v in ${VARIANTS:--}; do
  e=$(echo "$v" | tr "," " "); [ "$v" = "-" ] && e=""
  env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BARGS} > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/ab.log
done
