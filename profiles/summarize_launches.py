"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel (and GEMM grid)."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return [r for r in csv.DictReader(io.StringIO("".join(lines))) if r.get("Metric Name") == "gpu__time_duration.sum"]


def main(path, top=40):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        kn = r["Kernel Name"]
        name = kn.split("(")[0].replace("(anonymous namespace)::", "").replace("ttb::", "")
        if "gemm_kernel" in kn:
            name = "gemm<" + kn.split("gemm_kernel<")[1].split(">")[0] + "> grid" + r["Grid Size"]
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(rows)}  total {tot / 1e6:.3f} ms (cold-cache, serialised)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  avg={v[1] / v[0] / 1e3:9.1f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
