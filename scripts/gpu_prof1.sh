python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mid_spread_tile|k_near|k_long_gather|k_mid_gather|k_long_spread_tile" -s 0 -c 5 -o gpurun_out/prof1 python scripts/profile_eval.py c5 1 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu1.log
