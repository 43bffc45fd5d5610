"""Host memory of one reference DistributedRun at the bench workload (diagnostic for the
replica count of bench.py's reference arm)."""
import os
import sys
import time

import numpy as np
import psutil

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle.bindings import RefRun  # noqa: E402
from paper_2405_04416_b200 import workloads  # noqa: E402

p = psutil.Process()
wl = workloads.weak(1)
o, d, gt, _ = workloads.make_rays(wl.cfg, 4096, wl.generator, seed=1)
r0 = p.memory_info().rss
t = time.perf_counter()
run = RefRun(wl.cfg, workloads.appearance_rows(wl.cfg.appearance_dim, 1))
print("init s", time.perf_counter() - t, "rss GB", (p.memory_info().rss - r0) / 1e9)
img = np.zeros(512, np.uint32)
for s in range(2):
    t = time.perf_counter()
    run.train_step(o[:512], d[:512], gt[:512].astype(np.float64), img, s)
    print("step s", time.perf_counter() - t, "rss GB", (p.memory_info().rss - r0) / 1e9)
print("avail GB", psutil.virtual_memory().available / 1e9, "nparams", run.nparams(0))
