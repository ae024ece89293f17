# ncu --set full of one kernel (regex $1) in one c5 evaluation; summary + raw csv + source page
cd $GRAFT_REPO_ROOT
K=${1:-k_zpass}; CFG=${2:-c5}; TAG=${3:-prof}
python scripts/profile_eval.py $CFG 1 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 0 -c 1 -o gpurun_out/$TAG python scripts/profile_eval.py $CFG 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu=$?
python scripts/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>&1
cat gpurun_out/${TAG}_summary.txt
