# c5 bench A/B of in-tree library builds (SOG_LIB), then the GPU suite on $TESTLIB: run via gpurun
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for l in ${LIBS:-libsog.so}; do
  SOG_LIB=$PWD/paper_2412_04595_b200/lib/$l timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e ${BARGS} > gpurun_out/ab_$l.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$l.log').read().strip().splitlines()[-1]);print('$l', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stages_ms'].items()}, d.get('clocks',{}).get('sm_mhz'))" || tail -3 gpurun_out/ab_$l.log
done
done
if [ -n "$TESTLIB" ]; then
  SOG_LIB=$PWD/paper_2412_04595_b200/lib/$TESTLIB timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ab_pytest.log
fi
