# mid spread variant sweep (SOG_SPREAD_MMA values) at c5 + parity subset with the default
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py -q -x -k "not full_size" 2>&1 | tail -2
for v in ${VARIANTS:-1 20 21 30 31 41 0}; do
SOG_SPREAD_MMA=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sv$v.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_sv$v.log').read().strip().splitlines()[-1]);print('v=$v', round(d['ms_per_step'],2), 'spread', round(d['stages_ms']['mid_spread'],3))" || tail -3 gpurun_out/bench_sv$v.log
done
