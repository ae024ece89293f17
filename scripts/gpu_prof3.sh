python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_near2|k_mid_gather" -s 0 -c 2 -o gpurun_out/prof3 python scripts/profile_eval.py c5 1 > gpurun_out/ncu3.log 2>&1; echo ncu=$?
