"""Which gradient entries carry the largest error relative to their sum of |contributions|
(tied oracle step)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.bindings import OracleRun
from paper_2405_04416_b200 import dg, workloads
from tests.helpers import app_rows, small_cfg, rel_l2, layout_arrays, params_for, tied_train_step

cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
o, d, gt, img = workloads.make_rays(cfg, 2048, "independent", seed=9)
for scale in (None, 0.5):
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0); ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    for g in range(2):
        p = params_for(cfg, g, table_scale=scale); ctx.set_params(g, p); orc.set_params(g, p)
    sg, so, ovr = tied_train_step(ctx, orc, o, d, gt, img, 0)
    g = 0
    m, _, _ = ctx.get_adam(g)
    gg = m.astype(np.float64) / 0.1; go = orc.grads(g); ab = orc.abs_grads(g)
    names = [f"lvl{l}" for l in range(16)] + ["dw0", "db0", "dw1", "db1", "cw0", "cb0", "cw1", "cb1", "cw2", "cb2"]
    for a, nm in zip(layout_arrays(cfg, g)[:26], names):
        sl = slice(a["offset"], a["offset"] + a["size"])
        if np.abs(go[sl]).max() == 0: continue
        e = np.abs(gg[sl] - go[sl]) / np.maximum(ab[sl], 1e-30)
        if np.mean(e > 1e-4) > 0.001:
            w = np.argsort(-e)[:4]
            cols = {"dw0": 32, "dw1": 64, "cw0": 47, "cw1": 64, "cw2": 64}.get(nm, 2)
            print(scale, nm, f"frac>1e-4 {np.mean(e > 1e-4):.3f}", [(int(i) // cols, int(i) % cols, f"e={e[i]:.1e} g={go[sl][i]:.2e} abs={ab[sl][i]:.2e} gpu={gg[sl][i]:.2e}") for i in w])
