python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python scripts/diag_parity.py c5 20000 > gpurun_out/diag5.log 2>&1; echo diag5=$?; tail -8 gpurun_out/diag5.log
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mid_spread_tile" -s 0 -c 1 -o gpurun_out/prof2 python scripts/profile_eval.py c5 1 > gpurun_out/ncu2.log 2>&1; echo ncu=$?
