"""Gradient parity by state with the oracle tied to the GPU's ReLU decisions (tests/helpers.py
tied_train_step): what remains after kink ties is the arithmetic error."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.bindings import OracleRun
from paper_2405_04416_b200 import dg, workloads
from tests.helpers import app_rows, small_cfg, rel_l2, layout_arrays, params_for, tied_train_step

def run(cfg, o, d, gt, img, label, table_scale=None, bias=0.0, tie=True):
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0); ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    for g in range(cfg.kx * cfg.ky):
        p = params_for(cfg, g, table_scale=table_scale)
        for a in layout_arrays(cfg, g):
            if a["kind"] in (2, 4) and a["size"] == 64:
                p[a["offset"]:a["offset"] + a["size"]] = bias
        ctx.set_params(g, p); orc.set_params(g, p)
    if tie:
        sg, so, ovr = tied_train_step(ctx, orc, o, d, gt, img, 0)
    else:
        sg = ctx.train_step(o, d, gt, img, step=0); so = orc.train_step(o, d, gt, img, 0); ovr = None
    le = max(abs(sg[k] - so[k]) / abs(so[k]) for k in ("loss_rgb", "loss_transmittance", "loss_distortion"))
    by = {}
    for g in range(cfg.kx * cfg.ky):
        m, _, _ = ctx.get_adam(g)
        gg = m.astype(np.float64) / 0.1; go = orc.grads(g); ab = orc.abs_grads(g)
        for a in layout_arrays(cfg, g):
            sl = slice(a["offset"], a["offset"] + a["size"])
            if np.abs(go[sl]).max() == 0: continue
            e = np.abs(gg[sl] - go[sl]) / np.maximum(ab[sl], 1e-30)
            b = by.setdefault(a["kind"], [0, 0, 0])
            b[0] = max(b[0], rel_l2(gg[sl], go[sl])); b[1] = max(b[1], np.quantile(e, 0.999)); b[2] = max(b[2], np.mean(e > 1e-4))
    print(f"{label:28s} tie={tie} ovr={ovr} loss_rel={le:.1e} " + " ".join(f"k{k}:rl2={v[0]:.1e},q999={v[1]:.1e},f>1e-4={v[2]:.1e}" for k, v in sorted(by.items())), flush=True)

cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
o, d, gt, img = workloads.make_rays(cfg, 2048, "independent", seed=9)
impl = os.environ.get("DG_MLP", "tc")
for tie in (False, True):
    run(cfg, o, d, gt, img, f"{impl} init", tie=tie)
    run(cfg, o, d, gt, img, f"{impl} init+bias1", bias=1.0, tie=tie)
    run(cfg, o, d, gt, img, f"{impl} trained", table_scale=0.5, tie=tie)
    run(cfg, o, d, gt, img, f"{impl} trained+bias1", table_scale=0.5, bias=1.0, tie=tie)
