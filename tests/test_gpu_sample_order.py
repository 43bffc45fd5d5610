"""The spatial sample order (kernels_order.cu: Morton-sorted samples for the encode passes and
the MLP tiles; chunked or per-sample; the encoding backward's warp-aggregated scatter on any
number of levels) and the paired copies of the one-to-one level tables (kernels_pairs.cu) are
schedules / layouts, not changes of arithmetic: every mode must give the march-order step's
losses, gradients and render.

Only the fp32 summation order of the gradient scatter (atomics, warp sums) differs, so losses
and renders agree to fp32 rounding and gradients to 1e-5 relative L2 per array.  The oracle
parity of the default path (ordered, paired) is the rest of the GPU suite.
"""
import numpy as np
import pytest

from paper_2405_04416_b200 import dg, workloads

from .helpers import app_rows, inject, layout_arrays, rel_l2, small_cfg

pytestmark = pytest.mark.gpu

MODES = {
    "march": {"DG_SAMPLE_ORDER": "0"},
    "ordered": {"DG_SAMPLE_ORDER": "2"},
    "ordered_samples": {"DG_SAMPLE_ORDER": "2", "DG_ORDER_CHUNK": "1"},
    "ordered_chunk5": {"DG_SAMPLE_ORDER": "2", "DG_ORDER_CHUNK": "5", "DG_ORDER_BITS": "3"},
    "ordered_agg_all": {"DG_SAMPLE_ORDER": "2", "DG_ENC_AGG": "0.01"},
    "ordered_sliced": {"DG_SAMPLE_ORDER": "2", "DG_ENC_BWD_MB": "1", "DG_ENC_FWD_MB": "1"},
    "march_unpaired": {"DG_SAMPLE_ORDER": "0", "DG_ENC_PAIRED": "0"},
    "ordered_unpaired": {"DG_SAMPLE_ORDER": "2", "DG_ENC_PAIRED": "0"},
}
ENV = ("DG_SAMPLE_ORDER", "DG_ENC_PAIRED", "DG_ENC_AGG", "DG_ORDER_BITS", "DG_ORDER_CHUNK", "DG_ENC_BWD_MB", "DG_ENC_FWD_MB")


def _run(cfg, mode, monkeypatch, batch, state_seed=0, occupancy_fraction=None):
    for k in ENV:
        monkeypatch.delenv(k, raising=False)
    for k, v in MODES[mode].items():
        monkeypatch.setenv(k, v)
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)
    ctx.set_appearance(app)
    inject(cfg, ctx, [], seed=state_seed, occupancy_fraction=occupancy_fraction, table_scale=0.5)
    o, d, gt, img = batch
    rgb, T, depth = ctx.render(o, d, app[0])
    stats = ctx.train_step(o, d, gt, img, step=0)
    grads = [ctx.get_adam(g)[0].astype(np.float64) / (1.0 - cfg.adam_beta1) for g in range(cfg.kx * cfg.ky)]
    ctx.close()
    return stats, grads, (rgb, T, depth)


@pytest.mark.parametrize("case", ["1x1", "2x2_partial"])
def test_order_modes_agree(case, monkeypatch):
    if case == "1x1":
        cfg = small_cfg(1, 1, table_log2=14, levels=16, nmax=512, divisor=64)
        occ = None
        gen = "drift"
    else:
        cfg = small_cfg(2, 2, table_log2=13, levels=8, nmax=256, divisor=128,
                        inner=((0.3, 0.25, 0.0), (1.6, 1.8, 0.8)), occ_res=24)
        occ = 0.6
        gen = "independent"
    batch = workloads.make_rays(cfg, 4096, gen, seed=21)
    ref_stats, ref_grads, ref_render = _run(cfg, "march", monkeypatch, batch, occupancy_fraction=occ)
    for mode in [m for m in MODES if m != "march"]:
        stats, grads, render = _run(cfg, mode, monkeypatch, batch, occupancy_fraction=occ)
        for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
            assert abs(stats[k] - ref_stats[k]) <= 1e-6 * max(abs(ref_stats[k]), 1e-9), (mode, k)
        assert stats["samples"] == ref_stats["samples"]
        for a, b in zip(render, ref_render):
            assert np.allclose(a, b, rtol=1e-6, atol=1e-7), (mode, np.abs(a - b).max())
        for g in range(cfg.kx * cfg.ky):
            for arr in layout_arrays(cfg, g):
                sl = slice(arr["offset"], arr["offset"] + arr["size"])
                if np.abs(ref_grads[g][sl]).max() == 0:
                    assert np.abs(grads[g][sl]).max() == 0, (mode, g, arr)
                    continue
                e = rel_l2(grads[g][sl], ref_grads[g][sl])
                assert e < 1e-5, (mode, g, arr, e)
