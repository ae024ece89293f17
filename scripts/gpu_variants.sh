# Variant bench lines at HEAD (TAG = r02h): same list as gpu_round.sh.
TAG=${TAG:-r02h}
mkdir -p gpurun_out
for v in "--window kb:20" "--window es:20" "--long-method direct:20" "--config c4:150" "--config c4 --precision fp32 --tol 1e-4:300" \
         "--config c4 --long-method direct:150" "--config c2 --tol 1e-4:800" "--config c2 --tol 1e-8:300" "--config c2 --tol 1e-12:150" \
         "--config c3:80" "--config s1:80" "--config s1 --window kb:80" "--config t2:100" "--config t4:150" "--config t4 --window kb:150"; do
  args=${v%:*}; steps=${v##*:}
  tag=$(echo "$args" | tr -d ' -' | tr '.' '_')
  timeout 120 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-e2e $args > gpurun_out/${TAG}_var_$tag.log 2>&1; echo "bench $args = $?"
done
