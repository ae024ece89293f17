# Final evidence at HEAD (TAG = r02h), most important first: main bench (the driver's command), reference arm, smoke,
# ncu launch list of c5, GPU test suite, ncu --set full of the c5 stage kernels.  Variants: see r02f / r02g.
TAG=${TAG:-r02h}
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo bench=$?; tail -n 1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo ref=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -n 2 gpurun_out/smoke.log
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_eval.py c5 2 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 700 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/${TAG}_pytest_gpu.log
python scripts/profile_eval.py c5 1 > gpurun_out/plain1.log 2>&1 && \
timeout 500 ncu --set full --clock-control none --import-source on -k regex:"k_near3|k_mid_gather_z|k_mid_spread_zm|k_long_gather_bc|k_long_spread_gemm|k_zpass_t|k_combine|k_rows|k_xfft" -s 0 -c 11 -o gpurun_out/${TAG}_full python scripts/profile_eval.py c5 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_summary.txt 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_ncu_full_details.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/${TAG}_full.ncu-rep gpurun_out/${TAG}_ncu_traffic.json ${TAG}_ncu_full_details.txt > /dev/null 2>&1; echo traffic=$?
rm -f gpurun_out/${TAG}_full.ncu-rep
