import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.bindings import OracleRun
from paper_2405_04416_b200 import dg, layout, workloads
for wf in (0, 1):
    cfg = workloads._box_config((2, 1, 1), 2, 1, 14, 64, levels=8, nmax=256)
    cfg.wire_f32 = wf
    app = workloads.appearance_rows(16, 1).astype(np.float32).astype(np.float64)
    o, d, gt, img = workloads.make_rays(cfg, 512, "independent", seed=7)
    ctx = dg.Context(cfg, device=0); orc = OracleRun(cfg, app); ctx.set_appearance(app)
    for g in range(2):
        p = layout.reference_like_init(cfg, g); ctx.set_params(g, p); orc.set_params(g, p)
    rgb, T, depth = ctx.render(o, d, app[0])
    rgb_r, T_r, depth_r = orc.eval_rays(o, d, app[0])
    e = np.abs(rgb - rgb_r).max(axis=1); i = int(np.argmax(e))
    ns, reg, te, tx = orc_m = (None, None, None, None)
    print("wire", wf, "rgb maxabs", e.max(), "ray", i, rgb[i], rgb_r[i], "T", T[i], T_r[i], "Tmax", np.abs(T - T_r).max(), "depth", np.abs(depth-depth_r).max())
    # train-mode partials for the same ray?
