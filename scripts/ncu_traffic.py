"""Per-launch DRAM traffic of the stage kernels from an ncu --set full report, as the JSON bench.py
reads (profiles/r0N_ncu_traffic.json).  Usage: python scripts/ncu_traffic.py rep.ncu-rep out.json tag"""
import csv
import io
import json
import subprocess
import sys

STAGES = {"near": "k_near3<", "mid_spread": "k_mid_spread_z", "mid_gather": "k_mid_gather_z<",
          "long_spread": "k_long_spread_gemm<", "long_gather": "k_long_gather_bc<", "mid_scale": "k_zpass_r<"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    rep, out, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    rd, wr, du = (hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"))
    res = {}
    for r in rows[2:]:
        name = r[ki].replace("void ", "")
        for stage, pat in STAGES.items():
            if pat in name.replace("sog::", "") and stage not in res:
                b = float(r[rd].replace(",", "")) * UNIT.get(units[rd], 1.0) + \
                    float(r[wr].replace(",", "")) * UNIT.get(units[wr], 1.0)
                res[stage] = {"kernel": name.split("(")[0][:40], "dram_bytes_per_launch": b,
                              "ncu_duration_ms": float(r[du].replace(",", "")) * TUNIT.get(units[du], 1.0),
                              "source": f"profiles/{tag} (ncu --set full, c5, 1 launch)"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
