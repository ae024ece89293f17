# copy one gpu_round.sh run (TAG) from gpurun_out/ into profiles/ (bench lines, variants, launches, ncu summaries)
TAG=${1:-r02}
cd "$(dirname "$0")/.."
tail -1 gpurun_out/${TAG}_bench.log > profiles/${TAG}_bench.json
tail -1 gpurun_out/${TAG}_bench_ref.log > profiles/${TAG}_bench_ref.json
: > profiles/${TAG}_bench_variants.jsonl
for f in gpurun_out/${TAG}_var_*.log; do tail -1 "$f" | grep '^{' >> profiles/${TAG}_bench_variants.jsonl; done
cp gpurun_out/${TAG}_launches.csv profiles/${TAG}_launches.csv
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv > profiles/${TAG}_launches.txt
cp gpurun_out/${TAG}_ncu_full_summary.txt gpurun_out/${TAG}_ncu_full_details.txt gpurun_out/${TAG}_ncu_traffic.json profiles/ 2>/dev/null
cp gpurun_out/${TAG}_pytest_gpu.log profiles/ 2>/dev/null
ls -la profiles/${TAG}_*
