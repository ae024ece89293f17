"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass) by CUDA source
line: warp-stall samples and executed warp instructions, top N lines.

Usage: ncu -i rep --page source --csv --kernel-name regex:K --print-source cuda,sass > k.csv
       python scripts/ncu_lines.py k.csv [topN]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    fname, hdr, agg = "?", None, {}
    tot_s = tot_i = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ii = hdr.index("Instructions Executed")
            continue
        if hdr is None or not r[0] or len(r) <= max(si, ii):   # SASS rows: counted in their source line
            continue
        try:
            s = float(r[si])
            n = float(r[ii])
        except ValueError:
            continue
        key = (fname, r[0], r[1][:90])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += s
        a[1] += n
        tot_s += s
        tot_i += n
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
    for (f, ln, src), (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
        print(f"{100 * s / max(tot_s, 1):5.1f}% samp {100 * n / max(tot_i, 1):5.1f}% inst  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()


def reasons(path, lines):
    """Stall-reason breakdown of the given source line numbers."""
    rows = list(csv.reader(open(path)))
    hdr = None
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] in lines and len(r) == len(hdr):
            cols = [(h, float(v)) for h, v in zip(hdr, r) if h.startswith("stall_") and "Not Issued" not in h
                    and v not in ("", "-")]
            cols = sorted(cols, key=lambda t: -t[1])[:6]
            print(r[0], r[1][:50], " ".join(f"{h[6:]}={v:.0f}" for h, v in cols))
