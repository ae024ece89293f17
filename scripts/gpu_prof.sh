# ncu --set full of the kernels matching $1 (first $2 launches) in one c5 evaluation: summary, details, source csv
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-k_near5}; C=${2:-1}; TAG=${3:-prof}; CFG=${4:-c5}
python scripts/profile_eval.py $CFG 1 > gpurun_out/${TAG}_plain.log 2>&1 || { tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 0 -c $C -o gpurun_out/$TAG python scripts/profile_eval.py $CFG 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu=$?
python scripts/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>&1
cat gpurun_out/${TAG}_summary.txt
rm -f gpurun_out/$TAG.ncu-rep
