mkdir -p gpurun_out
for v in "--window kb:20" "--config c2 --tol 1e-4:800" "--config c2 --tol 1e-8:300" "--config c2 --tol 1e-12:150" "--config t4:150" "--config t4 --window kb:150"; do
  args=${v%:*}; steps=${v##*:}
  tag=$(echo "$args" | tr -d ' -' | tr '.' '_')
  timeout 600 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-e2e $args > gpurun_out/z_var_$tag.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/z_var_$tag.log').read().strip().splitlines()[-1]);print('$args', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()}, d['clocks'].get('sm_mhz'))" || tail -3 gpurun_out/z_var_$tag.log
done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/z_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/z_pytest.log
