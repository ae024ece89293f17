python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python scripts/diag_parity.py c1 1000 > gpurun_out/diag.log 2>&1; echo diag=$?; tail -9 gpurun_out/diag.log
timeout 1500 python -m pytest tests -q -m gpu -k "not c3_c4" --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench.log
