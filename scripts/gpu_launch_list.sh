# usage: CONF=s1 bash scripts/gpu_launch_list.sh <tag>   -- per-launch durations of one evaluation (ncu, serialised)
python scripts/profile_eval.py ${CONF:-c5} 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python scripts/profile_eval.py ${CONF:-c5} 1 > gpurun_out/ncu_ll_$1.log 2>&1; echo ncu=$?
