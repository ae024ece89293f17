# usage: bash scripts/gpu_prof_k.sh <kernel regex> <tag>
python scripts/profile_eval.py c5 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 0 -c 2 -o gpurun_out/prof_$2 python scripts/profile_eval.py c5 1 > gpurun_out/ncu_$2.log 2>&1; echo ncu=$?
