# Round evidence: smoke, GPU tests, full bench (CPU baseline + e2e), variant benches, ncu launch list,
# full capture of the top kernels summarised on the box (the report itself stays there: > 64 MiB)
mkdir -p gpurun_out
python -c "import paper_2412_04595_b200 as p; p.load_library()" > gpurun_out/build.log 2>&1; echo load=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -q -m gpu --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_full.log
for v in "--window kb" "--long-method direct" "--config c4" "--config c4 --precision fp32 --tol 1e-4" "--config c4 --long-method direct" \
         "--config c2 --tol 1e-4" "--config c2 --tol 1e-8" "--config c2 --tol 1e-12" "--config c3" "--config s1" "--config s1 --window kb" "--window es" \
         "--config t2" "--config t4" "--config t4 --window kb" "--config c5 --optimize"; do
  tag=$(echo "$v" | tr -d ' -' | tr '.' '_')
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $v > gpurun_out/bench_var_$tag.log 2>&1; echo "bench $v = $?"
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_near3|k_mid_gather_z|k_mid_spread_z|k_long_gather_bc|k_long_spread_gemm|k_tr_xz|k_scale_pencil_z" -s 0 -c 7 -o /tmp/prof_round python scripts/profile_eval.py c5 1 > gpurun_out/ncu_round.log 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py /tmp/prof_round.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
ncu -i /tmp/prof_round.ncu-rep --page details > gpurun_out/ncu_full_details.txt 2>&1
python scripts/ncu_traffic.py /tmp/prof_round.ncu-rep gpurun_out/ncu_traffic.json r01_ncu_full_v7.txt > /dev/null 2>&1; echo traffic=$?
