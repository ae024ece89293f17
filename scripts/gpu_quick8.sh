# parity (small) + c5 bench stage times; optional env for the bench in $BENV
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py -q -x -k "not full_size" 2>&1 | tail -2
env $BENV python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q8.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_q8.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/bench_q8.log
