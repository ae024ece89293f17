"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

Usage: python scripts/launch_summary.py gpurun_out/launches.csv [skip_first_n_launches]
Prints per kernel: launches, total / mean device time and share of the listed total.  ncu
serialises launches and runs them cold-cache: compare shares, not absolute times."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        out.append((r[ki], v * scale))
    return out


def main():
    launches = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    launches = launches[skip:]
    agg = collections.OrderedDict()
    for k, ms in launches:
        name = k.split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"{len(launches)} launches, {tot:.3f} ms total")
    print(f"{'kernel':60s} {'n':>5s} {'total ms':>10s} {'mean ms':>9s} {'share':>7s}")
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {n:5d} {ms:10.3f} {ms / n:9.4f} {100 * ms / tot:6.1f}%")


if __name__ == "__main__":
    main()
