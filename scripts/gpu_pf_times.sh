# per-kernel times of the plane FFT kernels (ncu launch list, one c5 evaluation per variant)
cd $GRAFT_REPO_ROOT
python scripts/profile_eval.py c5 1 > /dev/null 2>&1
for v in ${VARIANTS:-"SOG_PLANEFFT_B=4" "SOG_PLANEFFT_B=8"}; do
  echo "== $v"
  env $(echo $v | tr "," " ") ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rows|k_xfft|regular_fft|vector_fft" --csv python scripts/profile_eval.py c5 1 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for r in rows[1:]: print('%-60s %s'%(r[ik][:60], r[iv]))
"
done
