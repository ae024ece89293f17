# usage: bash scripts/gpu_prof_csv.sh <kernel regex> <tag>   (exports raw + source CSV on the box, keeps the report if small)
python scripts/profile_eval.py ${CONF:-c5} 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 0 -c 1 -o /tmp/prof_$2 python scripts/profile_eval.py ${CONF:-c5} 1 > gpurun_out/ncu_$2.log 2>&1; echo ncu=$?
ncu -i /tmp/prof_$2.ncu-rep --page raw --csv > gpurun_out/prof_$2_raw.csv 2>/dev/null
ncu -i /tmp/prof_$2.ncu-rep --page source --csv > gpurun_out/prof_$2_src.csv 2>/dev/null
ncu -i /tmp/prof_$2.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_$2_cuda.csv 2>/dev/null
ncu -i /tmp/prof_$2.ncu-rep --page details > gpurun_out/prof_$2_details.txt 2>/dev/null
ls -la gpurun_out/prof_$2*
