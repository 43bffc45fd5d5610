"""§8f row 4 (eval extras) on the GPU: dg_render_image (evaluate_image, worker.cpp:836-880)
against the oracle restatement, which tests/test_oracle_vs_reference.py pins bitwise to the
reference: colour / T / depth / region attribution within the forward bar (1e-4), with and
without the driver's early termination (worker.cpp:815-818)."""
import numpy as np
import pytest

from oracle.bindings import OracleRun
from paper_2405_04416_b200 import dg

from .helpers import app_rows, inject, small_cfg
from .test_oracle_vs_reference import _camera_rays, eval_camera

pytestmark = pytest.mark.gpu


def _close(a, b, rtol=1e-4, atol=2e-6):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert np.allclose(a, b, rtol=rtol, atol=atol), np.abs(a - b).max()


def test_render_image_matches_oracle():
    outs = {}
    for early in (0, 1):
        cfg = small_cfg(2, 2, table_log2=12, levels=6, nmax=128, divisor=48, occ_res=16)
        cfg.eval_early_termination = early
        cfg.eval_termination_threshold = 0.6
        app = app_rows(1)
        ctx = dg.Context(cfg, device=0)
        ctx.set_appearance(app.astype(np.float32))
        orc = OracleRun(cfg, app)
        inject(cfg, ctx, [orc], table_scale=0.5)
        cam = eval_camera()
        rgb, T, depth, attr = ctx.render_image(cam, app[0].astype(np.float32))
        o, d = _camera_rays(cam)
        r_rgb, r_T, r_depth, r_attr = orc.eval_rays_attribution(o, d, app[0])
        _close(rgb, r_rgb)
        _close(T, r_T)
        _close(depth, r_depth)
        _close(attr, r_attr)
        # the same rays through dg_render with an attribution output
        g = ctx.render(o, d, app[0].astype(np.float32), attribution=True)
        _close(g[3], r_attr)
        outs[early] = (T, depth)
    assert not np.array_equal(outs[0][1], outs[1][1])  # termination cut some rays short
