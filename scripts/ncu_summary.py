"""One-line-per-kernel summary of an ncu --set full report (duration, DRAM bytes, FP64 pipe,
issue, occupancy, shared-memory wavefronts).  Usage: python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cyc_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
}


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m in WANT if m in hdr}
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        vals = {}
        for m, i in idx.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if m == "gpu__time_duration.sum":
                v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1.0)
            if m.startswith("dram__bytes"):
                v *= {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1e-9)
            vals[WANT[m]] = v
        name = r[ki].split("(")[0].replace("void ", "")[:34]
        print(f"{name:34s} " + " ".join(f"{k}={v:.4g}" for k, v in vals.items()))


if __name__ == "__main__":
    main()
