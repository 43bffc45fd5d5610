"""Worst per-sample d_features errors of a training step (dg_last_sample_data vs the oracle's
sample log) and whether the forward's ReLU masks agree with the fp64 signs there: every large
error found so far is a mask tie at |z| <= ~1e-6 (tests/helpers.py tied_train_step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from oracle.bindings import gpu_mask_words
from tests.helpers import small_cfg
from tests.test_gpu_sample_parity import _run

for state in ("init", "trained", "trained+bias1"):
    cfg = small_cfg(2, 1, table_log2=14, levels=16, nmax=512, divisor=128)
    ctx, orc, (o, d, gt, img) = _run(cfg, 2048, "independent", 9, state)
    orc.log_samples(0, 4_000_000)
    ctx.train_step(o, d, gt, img, step=0)
    orc.train_step(o, d, gt, img, 0)
    pos, x, out, up, dx, mk = ctx.last_sample_data(0, masks=True)
    _, _, _, _, dx_o = orc.sample_log()
    wo, margin = orc.sample_log_masks()
    bad = (gpu_mask_words(mk) != wo).any(axis=1)
    e = np.abs(dx - dx_o).max(1) / np.maximum(np.abs(dx_o).max(1), 1e-30)
    print(state, "samples with a mask mismatch:", np.nonzero(bad)[0][:10], "of", len(bad))
    for w in np.argsort(-e)[:4]:
        print(f"  s{w} err {e[w]:.2e} mask mismatch {bad[w]} smallest |z| h1/c1/c2 {margin[w]}")
