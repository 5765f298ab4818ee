"""HBM-bound kernels of an ncu --set full capture: duration, DRAM bytes, achieved GB/s and its fraction
of the HBM peak (MEASURED_PEAKS.json hbm_gbs when the driver wrote it, else the B200_PROFILING.md
fallback 6650 GB/s). Usage: python profiles/hbm_summary.py report.ncu-rep [...]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        if "hbm_gbs" in j:
            return float(j["hbm_gbs"]), "MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for v in r[2:]:
        yield {h: (v[i], units[i]) for i, h in enumerate(hdr)}


def scale(val, unit):
    f = float(val)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)


if __name__ == "__main__":
    pk, src = peak()
    print(f"HBM peak {pk:.0f} GB/s ({src})")
    for path in sys.argv[1:]:
        for r in rows(path):
            name = r["Kernel Name"][0].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            t = scale(*r["gpu__time_duration.sum"])
            rd = scale(*r["dram__bytes_read.sum"])
            wr = scale(*r["dram__bytes_write.sum"])
            gbs = (rd + wr) / t / 1e9
            grid = r["Grid Size"][0]
            print(f"{name:40s} grid {grid:14s} {t * 1e6:9.1f} us  DRAM read {rd / 1e6:8.1f} MB  write {wr / 1e6:8.1f} MB"
                  f"  {gbs:7.0f} GB/s = {gbs / pk:5.2f} of peak   ({os.path.basename(path)})")
