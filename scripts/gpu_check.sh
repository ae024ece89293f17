# full GPU suite + smoke + c5 bench (stage times); the routine check after a change
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
env $BENV timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_check.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_check.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], {k:round(v,2) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/bench_check.log
