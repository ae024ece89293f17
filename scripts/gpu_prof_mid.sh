python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mid_spread_z|k_mid_gather_z" -s 0 -c 2 -o gpurun_out/prof_mid python scripts/profile_eval.py c5 1 > gpurun_out/ncu_mid.log 2>&1; echo ncu=$?
