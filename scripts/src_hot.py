"""Hot spots of an ncu --page source --csv export: per-opcode totals and the top stall lines.
Usage: python scripts/src_hot.py source.csv [ntop]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
R = rows[2:]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
iS, iw, ii, ist = (h.index(k) for k in ("Source", "L1 Wavefronts Shared", "Instructions Executed",
                                         "Warp Stall Sampling (All Samples)"))
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg = {}
tot = [0.0, 0.0, 0.0]
for r in R:
    try:
        w, n, st = float(r[iw] or 0), float(r[ii] or 0), float(r[ist] or 0)
    except ValueError:
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    a = agg.setdefault(op, [0, 0, 0])
    a[0] += w; a[1] += n; a[2] += st
    tot[0] += w; tot[1] += n; tot[2] += st
print("total: smem wf %.3g  inst %.3g  stall samples %d" % tuple(tot))
for k, v in sorted(agg.items(), key=lambda x: -x[1][2])[:15]:
    print("%-22s wf %.3g inst %.3g stall %d (%.1f%%)" % (k, v[0], v[1], v[2], 100 * v[2] / max(tot[2], 1)))
print("--- top lines by stall")
R2 = [r for r in R if len(r) > ist and r[ist].replace('.', '').isdigit()]
for r in sorted(R2, key=lambda r: -float(r[ist]))[:ntop]:
    reasons = sorted(((float(r[i] or 0), c[6:]) for i, c in stall_cols), reverse=True)[:3]
    print("%6s %-60s %s" % (r[ist], r[iS][:60], " ".join("%s:%d" % (c, v) for v, c in reasons if v)))
