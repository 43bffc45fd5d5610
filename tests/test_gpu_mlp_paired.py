"""The paired MLP backward for ReLU fields (kernels_mlp_tc.cu: k_mlp_bwd_tc_relu, the
input-gradient chain beside the forward recompute) is a schedule of the same GEMMs as the
serial kernel (k_mlp_bwd_tc, which the sigmoid / coarse fields keep): with
DG_MLP_BWD_SERIAL=1 every tile takes the serial kernel, and both must give the same losses,
render and gradients.

Only the fp32 summation order of the per-CTA weight-gradient flushes differs (the CTAs' tile
ranges change when the fine and coarse tiles are launched separately), so losses and renders
agree to fp32 rounding and gradients to 1e-5 relative L2 per array.  The oracle parity of the
default (paired) path is the rest of the GPU suite.
"""
import numpy as np
import pytest

from paper_2405_04416_b200 import dg, workloads

from .helpers import app_rows, inject, layout_arrays, rel_l2, small_cfg

pytestmark = pytest.mark.gpu


def _run(cfg, serial, monkeypatch, batch, occupancy_fraction=None):
    if serial:
        monkeypatch.setenv("DG_MLP_BWD_SERIAL", "1")
    else:
        monkeypatch.delenv("DG_MLP_BWD_SERIAL", raising=False)
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)
    ctx.set_appearance(app)
    inject(cfg, ctx, [], seed=0, occupancy_fraction=occupancy_fraction, table_scale=0.5)
    o, d, gt, img = batch
    rgb, T, depth = ctx.render(o, d, app[0])
    stats = ctx.train_step(o, d, gt, img, step=0)
    stats["coarse_samples"] = sum(int(ctx.last_items(g)[2]) for g in range(cfg.kx * cfg.ky))
    grads = [ctx.get_adam(g)[0].astype(np.float64) / (1.0 - cfg.adam_beta1) for g in range(cfg.kx * cfg.ky)]
    ctx.close()
    return stats, grads, (rgb, T, depth)


@pytest.mark.parametrize("case", ["1x1_fine_only", "2x2_fine_and_coarse"])
def test_paired_backward_matches_serial(case, monkeypatch):
    if case == "1x1_fine_only":
        cfg = small_cfg(1, 1, table_log2=14, levels=16, nmax=512, divisor=64)
        occ, gen = None, "drift"
    else:  # an inner (fine) box: every partition has fine (ReLU) and coarse (sigmoid) samples
        cfg = small_cfg(2, 2, table_log2=13, levels=8, nmax=256, divisor=128,
                        inner=((0.3, 0.25, 0.0), (1.6, 1.8, 0.8)), occ_res=24)
        occ, gen = 0.6, "independent"
    batch = workloads.make_rays(cfg, 4096, gen, seed=21)
    ref_stats, ref_grads, ref_render = _run(cfg, True, monkeypatch, batch, occupancy_fraction=occ)
    stats, grads, render = _run(cfg, False, monkeypatch, batch, occupancy_fraction=occ)
    assert (stats["coarse_samples"] > 0) == (case != "1x1_fine_only")
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(stats[k] - ref_stats[k]) <= 1e-6 * max(abs(ref_stats[k]), 1e-9), k
    assert stats["samples"] == ref_stats["samples"]
    for a, b in zip(render, ref_render):  # the render forward does not use the backward: identical
        assert np.array_equal(a, b)
    for g in range(cfg.kx * cfg.ky):
        for arr in layout_arrays(cfg, g):
            sl = slice(arr["offset"], arr["offset"] + arr["size"])
            if np.abs(ref_grads[g][sl]).max() == 0:
                assert np.abs(grads[g][sl]).max() == 0, (g, arr)
                continue
            e = rel_l2(grads[g][sl], ref_grads[g][sl])
            assert e < 1e-5, (g, arr, e)
