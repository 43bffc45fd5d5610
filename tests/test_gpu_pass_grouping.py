"""Encode pass grouping with large hashed tables (runtime.cu field_launch): passes that hold a
hashed table of >= 8 MB group levels only up to 64 MB forward / 32 MB backward
(DG_ENC_FWD_HGROUP_MB / DG_ENC_BWD_HGROUP_MB; BASELINE C2 has 32 MB hashed levels).  Grouping
is a schedule, not a change of arithmetic: every level is still encoded and scattered exactly
once, so the default and the ungrouped (0: the 192 / 96 MB budgets) runs give the same losses
and render to fp32 rounding and the same gradients to 1e-5 relative L2 per array.  The
oracle parity of the encode itself is the rest of the GPU suite (small tables, one pass) and
test_gpu_full_size.py (C4 and C1 grids, sliced passes).
"""
import numpy as np
import pytest

from paper_2405_04416_b200 import dg, workloads

from .helpers import app_rows, layout_arrays, rel_l2, small_cfg

pytestmark = pytest.mark.gpu

KNOBS = ("DG_ENC_FWD_HGROUP_MB", "DG_ENC_BWD_HGROUP_MB")


def _run(cfg, env, monkeypatch, batch):
    for k in KNOBS:
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)
    ctx.init_fast(0, seed=1)
    ctx.set_appearance(app)
    o, d, gt, img = batch
    render = ctx.render(o, d, app[0])
    stats = ctx.train_step(o, d, gt, img, step=0)
    grads = ctx.get_adam(0)[0].astype(np.float64) / (1.0 - cfg.adam_beta1)
    ctx.close()
    return stats, grads, render


def test_hashed_pass_grouping_is_a_schedule(monkeypatch):
    # T = 2^22: 32 MB hashed levels (levels 7-15), as in BASELINE C2
    cfg = small_cfg(1, 1, table_log2=22, levels=16, nmax=2048, divisor=64)
    batch = workloads.make_rays(cfg, 8192, "drift", seed=5)
    ref_stats, ref_grads, ref_render = _run(cfg, {k: "0" for k in KNOBS}, monkeypatch, batch)
    stats, grads, render = _run(cfg, {}, monkeypatch, batch)
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(stats[k] - ref_stats[k]) <= 1e-6 * max(abs(ref_stats[k]), 1e-9), k
    assert stats["samples"] == ref_stats["samples"]
    for a, b in zip(render, ref_render):
        assert np.allclose(a, b, rtol=1e-6, atol=1e-7), np.abs(a - b).max()
    checked = 0
    for arr in layout_arrays(cfg, 0):
        sl = slice(arr["offset"], arr["offset"] + arr["size"])
        if np.abs(ref_grads[sl]).max() == 0:
            assert np.abs(grads[sl]).max() == 0, arr
            continue
        e = rel_l2(grads[sl], ref_grads[sl])
        assert e < 1e-5, (arr, e)
        checked += 1
    assert checked > 16
