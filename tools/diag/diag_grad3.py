import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.bindings import OracleRun
from paper_2405_04416_b200 import dg, workloads
from tests.helpers import app_rows, inject, small_cfg, rel_l2, layout_arrays
cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
o, d, gt, img = workloads.make_rays(cfg, 2048, "independent", seed=9)
app = app_rows(1)
ctx = dg.Context(cfg, device=0); ctx.set_appearance(app)
orc = OracleRun(cfg, app)
inject(cfg, ctx, [orc])
sg = ctx.train_step(o, d, gt, img, step=0); so = orc.train_step(o, d, gt, img, 0)
print({k: (sg[k], so[k]) for k in ("loss_rgb", "loss_transmittance", "loss_distortion")})
for g in range(2):
    m, _, _ = ctx.get_adam(g)
    gg = m.astype(np.float64) / 0.1; go = orc.grads(g); ab = orc.abs_grads(g)
    errs = []
    for a in layout_arrays(cfg, g):
        sl = slice(a["offset"], a["offset"] + a["size"])
        if np.abs(go[sl]).max() > 0: errs.append("%.1e" % rel_l2(gg[sl], go[sl]))
    print("part", g, errs)
    sl = slice(0, 8192)
    diff = np.abs(gg[sl] - go[sl]); idx = np.argsort(-diff)[:12]
    for k in idx:
        row, f = divmod(int(k), 2); ix, r2 = row % 16, row // 16; iy, iz = r2 % 16, r2 // 16
        print("  l0 entry", k, (ix, iy, iz, f), "gpu %.6e ref %.6e abs %.3e diff %.3e" % (gg[k], go[k], ab[k], diff[k]))
