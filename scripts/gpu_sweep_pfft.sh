# plane-FFT check: parity subset + c5 bench for SOG_PLANEFFT / SOG_PLANEFFT_B variants
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kb.py -q -x -k "not full_size" 2>&1 | tail -2
for v in ${VARIANTS:-"SOG_PLANEFFT=0" "SOG_PLANEFFT_B=8" "SOG_PLANEFFT_B=4" "SOG_PLANEFFT_B=16"}; do
env $(echo $v | tr "," " ") python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_pf.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_pf.log').read().strip().splitlines()[-1]);s=d['stages_ms'];print('$v', round(d['ms_per_step'],2), 'fwd', round(s['mid_fft_fwd'],3), 'inv', round(s['mid_fft_inv'],3), 'zpass', round(s['mid_scale'],3))" || tail -3 gpurun_out/bench_pf.log
done
