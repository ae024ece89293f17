cd $GRAFT_REPO_ROOT
python scripts/diag_stages.py c2 3000 1e-12 gs,kb,es
SOG_ZPASS=0 python scripts/diag_stages.py c2 3000 1e-12 gs,kb
python scripts/diag_stages.py s1 3000 1e-12 gs,kb
python scripts/diag_stages.py c1 1000 1e-6 gs,kb
python -m pytest tests/test_gpu_parity.py -q -k "c1_ or c2_tol or shapes_small" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_zpass.log 2>&1; tail -1 gpurun_out/bench_zpass.log
SOG_ZPASS=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_nozpass.log 2>&1; tail -1 gpurun_out/bench_nozpass.log
./scripts/bin/fp64_peak 60 > gpurun_out/fp64_peak2.txt 2>&1
