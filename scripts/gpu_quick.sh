# quick check: c1 stage parity + c5 bench (zpass on / off)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -q -k "c1_ or c2_tol or shapes_small or edge" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q1.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_q1.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['stages_ms'])"
