"""Bisect the level-0 gradient mismatch of test_train_step_parity[2-1-independent-2048-init]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.bindings import OracleRun, OracleModel
from paper_2405_04416_b200 import dg, workloads
from tests.helpers import app_rows, inject, small_cfg, rel_l2, layout_arrays

cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
o, d, gt, img = workloads.make_rays(cfg, 2048, "independent", seed=9)
ns, reg, te, tx = OracleModel(cfg).segment_rays(o, d)

def run(sel, label):
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0); ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    inject(cfg, ctx, [orc])
    sg = ctx.train_step(o[sel], d[sel], gt[sel], img[sel], step=0); so = orc.train_step(o[sel], d[sel], gt[sel], img[sel], 0)
    out = []
    for g in range(2):
        m, _, _ = ctx.get_adam(g)
        gg = m.astype(np.float64) / 0.1
        go = orc.grads(g)
        a = layout_arrays(cfg, g)[0]
        sl = slice(a["offset"], a["offset"] + a["size"])
        out.append(rel_l2(gg[sl], go[sl]))
    print(label, len(sel), ["%.2e" % x for x in out], flush=True)
    return max(out)

allr = np.arange(len(o))
run(allr, "all")
run(allr[ns == 1], "single")
run(allr[ns == 2], "double")
# bisect over multi-segment rays if they carry the error
cand = allr[ns == 2] if run(allr[ns == 2], "double") > 1e-4 else allr
while len(cand) > 1:
    h = len(cand) // 2
    a, b = cand[:h], cand[h:]
    ea = run(a, "A"); eb = run(b, "B")
    if ea >= eb: cand = a
    else: cand = b
    if max(ea, eb) < 1e-5: break
print("culprit rays", cand[:10])
for i in cand[:3]:
    print(i, o[i].tolist(), d[i].tolist(), ns[i], reg[i, :ns[i]].tolist(), te[i, :ns[i]].tolist(), tx[i, :ns[i]].tolist())
