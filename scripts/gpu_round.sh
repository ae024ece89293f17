# Round evidence (run on the GPU box via gpurun): GPU test suite, smoke, main bench (the driver's command), reference
# arm, variant benches (each timed region >= ~0.5 s), ncu launch list of one c5 evaluation, ncu --set
# full of the stage kernels of one c5 evaluation (summary, traffic table, details).  TAG = r02.
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo ref=$?
for v in "--window kb:20" "--window es:20" "--long-method direct:20" "--config c4:150" "--config c4 --precision fp32 --tol 1e-4:300" \
         "--config c4 --long-method direct:150" "--config c2 --tol 1e-4:800" "--config c2 --tol 1e-8:300" "--config c2 --tol 1e-12:150" \
         "--config c3:80" "--config s1:80" "--config s1 --window kb:80" "--config t2:100" "--config t4:150" "--config t4 --window kb:150"; do
  args=${v%:*}; steps=${v##*:}
  tag=$(echo "$args" | tr -d ' -' | tr '.' '_')
  timeout 600 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-e2e $args > gpurun_out/${TAG}_var_$tag.log 2>&1; echo "bench $args = $?"
done
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_eval.py c5 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/profile_eval.py c5 1 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_near3|k_mid_gather_z|k_mid_spread_zm|k_long_gather_bc|k_long_spread_gemm|k_zpass_t|k_combine|k_rows|k_xfft" -s 0 -c 11 -o gpurun_out/${TAG}_full python scripts/profile_eval.py c5 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_summary.txt 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_ncu_full_details.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/${TAG}_full.ncu-rep gpurun_out/${TAG}_ncu_traffic.json ${TAG}_ncu_full_details.txt > /dev/null 2>&1; echo traffic=$?
rm -f gpurun_out/${TAG}_full.ncu-rep
