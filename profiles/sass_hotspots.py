"""Per-SASS-line stall samples of an ncu --set full report (--page source), grouped into the
contiguous instruction ranges between two given line numbers, with the stall-reason breakdown.
Usage: python profiles/sass_hotspots.py report.ncu-rep [top N]"""
import csv
import io
import subprocess
import sys


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[1], rows[2:]


def main(path, top=40):
    hdr, R = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in R)
    print(f"total stall samples {tot}")
    lines = []
    for n, r in enumerate(R):
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        if s:
            rs = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
            lines.append((s, n, r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0), rs))
    for s, n, src, ex, rs in sorted(lines, reverse=True)[:top]:
        print(f"{s:7d} {100 * s / tot:5.1f}%  L{n:<5d} x{ex:<9d} {src[:70]:70s} " + " ".join(f"{h}={v}" for v, h in rs if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
