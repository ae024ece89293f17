# Round evidence: smoke, GPU tests, full bench (CPU baseline + e2e), ncu launch list, full capture of the top kernels
python -c "import paper_2412_04595_b200 as p; p.load_library()" > gpurun_out/build.log 2>&1; echo load=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_full.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_near3|k_mid_gather_z|k_mid_spread_z|k_long_gather_bc|k_long_spread_gemm|k_tr_xz|k_scale_pencil_z" -s 0 -c 7 -o gpurun_out/prof_round python scripts/profile_eval.py c5 1 > gpurun_out/ncu_round.log 2>&1; echo ncu_full=$?
