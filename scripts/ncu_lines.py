"""Aggregate ncu source-page (cuda,sass) CSV by CUDA source line: stall samples and instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = next(i for i, r in enumerate(rows) if any('Sampling' in c for c in r))
hdr = rows[hdr_i]
si = hdr.index('Warp Stall Sampling (All Samples)'); ii = hdr.index('Instructions Executed')
agg = collections.defaultdict(lambda: [0, 0])
cur = None
tot_s = tot_i = 0
for r in rows[hdr_i + 1:]:
    if len(r) < 5:
        continue
    if r[0]:
        cur = (r[0], r[1][:100])
    try:
        s = float(r[si] or 0); n = float(r[ii] or 0)
    except ValueError:
        continue
    if cur:
        agg[cur][0] += s; agg[cur][1] += n
    tot_s += s; tot_i += n
print(f"total samples {tot_s:.0f} instructions {tot_i:.3e}")
for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
    print(f"{100*s/max(tot_s,1):5.1f}% samp {100*n/max(tot_i,1):5.1f}% inst  L{k[0]}  {k[1]}")
