# dev loop: parity diagnostics, GPU tests, short bench
python -c "import paper_2412_04595_b200 as p; p.load_library()" > gpurun_out/build.log 2>&1; echo load=$?
timeout 300 python scripts/diag_parity.py c1 1000 > gpurun_out/diag.log 2>&1; echo diag=$?; tail -9 gpurun_out/diag.log
timeout 300 python scripts/diag_parity.py c5 20000 > gpurun_out/diag5.log 2>&1; echo diag5=$?; tail -9 gpurun_out/diag5.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], {k:round(v,2) for k,v in d['stages_ms'].items()})"
