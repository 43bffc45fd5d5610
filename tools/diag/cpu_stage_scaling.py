"""Thread scaling of the reference stage functions on this host (diagnostic for bench.py's
cpu_stages baseline)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle.bindings import RefRun  # noqa: E402
from paper_2405_04416_b200 import workloads  # noqa: E402

wl = workloads.weak(1, rays_per_gpu=4096, table_log2=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
o, d, _, _ = workloads.make_rays(wl.cfg, 32768, wl.generator, seed=1)
run = RefRun(wl.cfg, workloads.appearance_rows(wl.cfg.appearance_dim, 1))
rng = np.random.default_rng(1)
pts = rng.uniform(size=(65536, 3))
dirs = rng.normal(size=(65536, 3))
dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
for th in (1, 2, 4, 8, 16):
    r = run.stage_bench(o, d, pts, dirs, th, 1)
    print(th, {k: round(v) for k, v in r.items()})
