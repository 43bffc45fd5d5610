"""Per-step wall/device times around the occupancy update (diagnostic).
Usage (GPU): python tools/step_timeline.py"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_04416_b200 import abi, dg, workloads  # noqa: E402

wl = workloads.weak(1)
cfg = wl.cfg
ctx = dg.Context(cfg, device=0)
ctx.init_fast(0, seed=1)
ctx.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))
o, d, gt, img = workloads.make_rays(cfg, wl.n_rays, wl.generator, seed=1)
t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (o, d, gt, img.astype(np.int32))]
b = abi.RayBatch()
b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), t[3].data_ptr())
b.n, b.first_ray_id, b.mem = len(o), 0, abi.DG_MEM_DEVICE
st = abi.StepStats()
ctx.enable_stage_timing(True)
for i in range(40):
    torch.cuda.synchronize()
    a = time.perf_counter()
    assert ctx.train_step_raw(b, i, st) == 0
    torch.cuda.synchronize()
    w = (time.perf_counter() - a) * 1e3
    tot = ctx.stage_times()["total"]
    print(f"step {i:3d} wall {w:7.2f} ms  device(marks) {tot:7.2f} ms  launches {ctx.kernel_launches()}"
          f"  samples {st.samples}")
    if i in (14, 20, 39):
        print("   stages:", {k: round(v, 3) for k, v in ctx.stage_times().items()})
