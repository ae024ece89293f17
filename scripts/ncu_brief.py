"""Brief ncu report digest: speed-of-light, occupancy, stall mix, instruction mix with lane activity.
usage: python scripts/ncu_brief.py TAG   (reads gpurun_out/TAG_details.txt and TAG_source.csv)"""
import collections
import csv
import re
import sys

tag = sys.argv[1]
for line in open(f"gpurun_out/{tag}_details.txt"):
    if re.search(r"Duration|Throughput|Issue Slots|Eligible Warps|Warp Cycles Per Issued|Theoretical Occ|Achieved Occ|"
                 r"Registers Per|bank|excessive", line):
        print(line.rstrip()[:150])
rows = list(csv.reader(open(f"gpurun_out/{tag}_source.csv")))
hdr = rows[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in rows[2:]:
    for i in cols:
        try:
            tot[hdr[i]] += float(r[i])
        except ValueError:
            pass
s = sum(tot.values())
print("stalls:", [(k[6:], round(v / s, 3)) for k, v in tot.most_common(8)])
ii, ti, si = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Source")
agg = collections.defaultdict(lambda: [0.0, 0.0])
for r in rows[2:]:
    try:
        v, t = float(r[ii]), float(r[ti])
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9]+)", r[si])
    if m:
        agg[m.group(2)][0] += v
        agg[m.group(2)][1] += t
T = sum(v[0] for v in agg.values())
print("warp instructions %.4g" % T)
print("mix:", [(k, round(v[0] / T, 3), round(v[1] / v[0], 1)) for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:16]])
