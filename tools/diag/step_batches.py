import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2405_04416_b200 import abi, dg, workloads
wl = workloads.weak(1); cfg = wl.cfg
ctx = dg.Context(cfg, device=0); ctx.init_fast(0, seed=1)
ctx.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))
bs = []
for k in range(3):
    o, d, gt, img = workloads.make_rays(cfg, wl.n_rays, wl.generator, seed=1 + k)
    t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (o, d, gt, img.astype(np.int32))]
    b = abi.RayBatch(); b.origin, b.dir, b.color_gt, b.image_id = (t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), t[3].data_ptr())
    b.n, b.first_ray_id, b.mem = len(o), 0, abi.DG_MEM_DEVICE
    bs.append((b, t))
st = abi.StepStats(); ctx.enable_stage_timing(True)
for i in range(int(os.environ.get("STEPS", "12"))):
    torch.cuda.synchronize(); a = time.perf_counter()
    assert ctx.train_step_raw(bs[i % 3][0], i, st) == 0
    torch.cuda.synchronize(); w = (time.perf_counter() - a) * 1e3
    stt = ctx.stage_times()
    print(f"step {i:2d} batch {i%3} wall {w:6.2f} device {stt['total']:6.2f}", {k: round(v, 2) for k, v in stt.items() if k in ("march", "encode_fwd", "mlp_fwd", "mlp_bwd", "encode_bwd", "adam")})
