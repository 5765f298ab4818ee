"""c5 sweep (BASELINE.json configs[4]): prefix-share ratio r in {0, 0.1, ..., 0.9} on the Qwen2-0.5B
shape, tree (DFS prefix-tree step) vs flat (same engine, every rollout its own root), 1 GPU, with the
per-point CPU reference extrapolation. Runs bench.py once per ratio and writes one JSON object.
Usage: python tools/sweep_c5.py [--prompts P] [--out gpurun_out/c5_sweep.json]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=8)
    ap.add_argument("--ratios", default="0,0.1,0.2,0.3,0.4,0.5,0.6,0.7,0.8,0.9")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5_sweep.json"))
    args = ap.parse_args()
    points = []
    for r in (float(x) for x in args.ratios.split(",")):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5", "--share", str(r), "--prompts",
               str(args.prompts), "--steps", "2", "--warmup", "3", "--no-e2e"]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        line = next((l for l in out.stdout.splitlines() if l.startswith("{")), None)
        if line is None:
            points.append({"share": r, "error": out.stderr[-2000:]})
            continue
        j = json.loads(line)
        points.append({"share": r, "duplication_factor": j["tree"]["duplication_factor"],
                       "tree_tokens_per_s": j["value"], "flat_tokens_per_s": j.get("flat", {}).get("value"),
                       "tree_over_flat": j["value"] / j["flat"]["value"] if j.get("flat") else None,
                       "tree_peak_hbm_gb": j["peak_hbm_gb"], "flat_peak_hbm_gb": j.get("flat", {}).get("peak_hbm_gb"),
                       "cpu_reference_tokens_per_s": j.get("cpu_baseline", {}).get("value"),
                       "ms_per_step": j["ms_per_step"], "clocks": j.get("clocks")})
        print(json.dumps(points[-1]), flush=True)
    res = {"config": f"c5: Qwen2-0.5B-shape, {args.prompts} prompts x 16 rollouts x 4096 tokens, shared prefix r*4096 "
                     "(weights 0) + response (weights 1), 1 B200; tree = DFS prefix-tree step, flat = same engine "
                     "with every rollout its own root", "unit": "rollout tokens/s", "points": points}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
