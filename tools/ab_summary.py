"""Summarise tools/ab_pair.sh output: tests, then per bench log the training rays/s, step and
MLP-backward stage times.  Usage: python tools/ab_summary.py gpurun_out/TAG"""
import glob
import json
import os
import sys

d = sys.argv[1]
print(open(os.path.join(d, "t1.log")).read().strip().splitlines()[-2:])
for f in sorted(glob.glob(os.path.join(d, "bench_*.log"))):
    for line in open(f):
        if line.startswith("{"):
            j = json.loads(line)
            st = j["roofline"]["stage_ms"]
            print(os.path.basename(f), f"{j['value'] / 1e6:.3f} M rays/s", f"{j['ms_per_step']:.3f} ms",
                  f"mlp_bwd {st['mlp_bwd']:.3f}", f"mlp_fwd {st['mlp_fwd']:.3f}",
                  f"render {j['render_rays_per_s'] / 1e6:.2f}")
        elif "rror" in line:
            print(os.path.basename(f), line.strip()[:300])
