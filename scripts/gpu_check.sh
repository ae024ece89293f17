# all GPU tests + smoke + short benches (fp64 c5 headline, fp32 c4)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
timeout 600 python bench.py --config c4 --precision fp32 --tol 1e-4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4f32.log 2>&1; echo bench32=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4f32.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4f64.log 2>&1; echo bench64c4=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_c4f64.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
