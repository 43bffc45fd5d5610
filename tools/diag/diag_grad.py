"""Diagnostic: where does the level-0 gradient mismatch of multi-partition steps come from?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.bindings import OracleRun, OracleModel
from paper_2405_04416_b200 import dg, workloads
from tests.helpers import app_rows, inject, small_cfg, rel_l2, layout_arrays

def run(cfg, o, d, gt, img, label):
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0); ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    inject(cfg, ctx, [orc])
    sg = ctx.train_step(o, d, gt, img, step=0); so = orc.train_step(o, d, gt, img, 0)
    print(label, {k: (sg[k], so[k]) for k in ("loss_rgb", "loss_transmittance", "loss_distortion")})
    for g in range(cfg.kx * cfg.ky):
        m, _, _ = ctx.get_adam(g)
        gg = m.astype(np.float64) / 0.1
        go = orc.grads(g); ab = orc.abs_grads(g)
        errs = []
        for a in layout_arrays(cfg, g)[:6]:
            sl = slice(a["offset"], a["offset"] + a["size"])
            errs.append((round(rel_l2(gg[sl], go[sl]), 7), round(np.linalg.norm(gg[sl]-go[sl]) / max(np.linalg.norm(ab[sl]), 1e-30), 7)))
        print("  part", g, errs)
        # worst entries of level 0
        sl = slice(0, layout_arrays(cfg, g)[0]["size"])
        diff = np.abs(gg[sl] - go[sl]); i = np.argsort(-diff)[:5]
        print("   worst l0 entries", [(int(k), float(gg[k]), float(go[k]), float(ab[k])) for k in i])

cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
o, d, gt, img = workloads.make_rays(cfg, 2048, "independent", seed=8)
run(cfg, o, d, gt, img, "2x1 independent")
ov, dv, gtv, imgv = workloads.make_rays(cfg, 2048, "vertical", seed=8)
run(cfg, ov, dv, gtv, imgv, "2x1 vertical (single-segment)")
cfg1 = small_cfg(1, 1, table_log2=14, levels=16, nmax=512, divisor=64)
o1, d1, gt1, img1 = workloads.make_rays(cfg1, 2048, "independent", seed=8)
run(cfg1, o1, d1, gt1, img1, "1x1 independent")
