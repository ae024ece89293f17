# quick check: parity subset + c5 bench stage times (near kernel variants via SOG_NEAR)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py tests/test_dist_gpu.py -q -x -k "c1_ or c2_tol or shapes_small or loopback or confined" 2>&1 | tail -3
for m in ${NEAR_MODES:-4 5}; do
SOG_NEAR=$m python -m pytest tests/test_gpu_parity.py -q -x -k "c1_ or c2_tol or shapes_small" 2>&1 | tail -1
SOG_NEAR=$m python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q$m.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_q$m.log').read().strip().splitlines()[-1]);print('near mode $m', d['ms_per_step'], d['stages_ms']['near'])" || tail -5 gpurun_out/bench_q$m.log
done
