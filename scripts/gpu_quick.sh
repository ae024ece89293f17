# quick check: parity subset + c5 bench stage times
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py tests/test_dist_gpu.py -q -x -k "c1_ or c2_tol or shapes_small or loopback or confined or fp32" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/bench_q.log
