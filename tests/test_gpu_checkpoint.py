"""§8f row 3: .dgcw checkpoint interop with the reference (checkpoint.cpp:241-283).

* identical state on both sides -> the GPU writer and the reference writer produce the same
  bytes;
* after a training step on each side, a reference-written checkpoint loads into the GPU
  context exactly (tables/MLPs as the file's f32, Adam moments as f32 of the file's f64,
  occupancy density, threshold, step) and a GPU-written checkpoint loads into the reference
  exactly (Worker::load_state);
* training continues from a loaded state in step with the reference.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle.bindings import RefRun, ref_available
from paper_2405_04416_b200 import dg, layout, workloads

from .helpers import app_rows, inject, rel_err, small_cfg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) missing")]

HASH = 0x1234_5678_9ABC_DEF0


def _setup():
    cfg = small_cfg(2, 1, table_log2=12, levels=8, nmax=128, divisor=96, occ_res=16)
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)
    ctx.set_appearance(app.astype(np.float32))
    ref = RefRun(cfg, app)
    inject(cfg, ctx, [ref], occupancy_fraction=0.7)
    return cfg, ctx, ref


def test_checkpoint_bytes_identical():
    cfg, ctx, ref = _setup()
    with tempfile.TemporaryDirectory() as td:
        for g in range(2):
            a, b = os.path.join(td, f"gpu{g}.dgcw"), os.path.join(td, f"ref{g}.dgcw")
            ctx.save_checkpoint(g, HASH, a)
            ref.save_checkpoint(g, HASH, b)
            ba, bb = open(a, "rb").read(), open(b, "rb").read()
            assert len(ba) == len(bb)
            assert ba == bb, next(i for i in range(len(ba)) if ba[i] != bb[i])


def test_checkpoint_round_trips_after_training():
    cfg, ctx, ref = _setup()
    o, d, gt, img = workloads.make_rays(cfg, 1500, "independent", seed=4)
    ctx.train_step(o, d, gt, img, step=0)
    ref.train_step(o, d, gt, img, 0)
    with tempfile.TemporaryDirectory() as td:
        # reference -> GPU
        fresh = dg.Context(cfg, device=0)
        fresh.set_appearance(app_rows(1).astype(np.float32))
        for g in range(2):
            path = os.path.join(td, f"ref{g}.dgcw")
            ref.save_checkpoint(g, HASH, path)
            assert fresh.load_checkpoint(g, path) == HASH
            assert np.array_equal(fresh.get_params(g), ref.params(g).astype(np.float32))
            m, v, t = fresh.get_adam(g)
            rm, rv, rt, _ = ref.adam(g)
            assert t == rt
            assert np.array_equal(m, rm.astype(np.float32)) and np.array_equal(v, rv.astype(np.float32))
            for c, box in enumerate(layout.region_boxes(cfg, g)):
                n = int(np.prod(layout.occupancy_shape(cfg, box)))
                assert np.array_equal(fresh.get_occupancy(g, c), ref.occupancy(g, c, n))
        assert fresh.get_step() == 1
        # GPU -> reference
        ref2 = RefRun(cfg, app_rows(1))
        for g in range(2):
            path = os.path.join(td, f"gpu{g}.dgcw")
            ctx.save_checkpoint(g, HASH, path)
            assert ref2.load_checkpoint(g, path) == HASH
            assert np.array_equal(ref2.params(g), ctx.get_params(g).astype(np.float64))
            m, v, t = ctx.get_adam(g)
            rm, rv, rt, _ = ref2.adam(g)
            assert t == rt and np.array_equal(rm, m.astype(np.float64)) and np.array_equal(rv, v.astype(np.float64))
        # training continues in step from the reference-written state
        o2, d2, gt2, img2 = workloads.make_rays(cfg, 1500, "independent", seed=9)
        sg = fresh.train_step(o2, d2, gt2, img2, step=1)
        sr = ref.train_step(o2, d2, gt2, img2, 1)
        for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
            assert rel_err(sg[k], sr[k], 1e-9) < 1e-4, (k, sg[k], sr[k])


def test_checkpoint_rejects_mismatch():
    cfg, ctx, ref = _setup()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "r0.dgcw")
        ref.save_checkpoint(0, HASH, path)
        with pytest.raises(dg.DGError):
            ctx.load_checkpoint(1, path)  # region mismatch (worker.cpp:616-617)
        with open(path, "r+b") as f:
            f.write(b"XXXX")
        with pytest.raises(dg.DGError):
            ctx.load_checkpoint(0, path)


def test_resume_past_warmup_keeps_occupancy_stream():
    """a fresh context draws the next warm-up update's jitter points ahead of time
    from its occupancy mt19937_64 stream.  Loading a checkpoint past the warm-up must rewind
    those draws, so the first sampled (non-warm-up) update after the resume takes the same
    cells and jitter points as the reference's fresh Worker after load_state
    (worker.cpp:549-562, 615-626)."""
    cfg = small_cfg(2, 1, table_log2=12, levels=8, nmax=128, divisor=64, occ_res=16,
                    inner=((0.2, 0.1, 0.0), (1.7, 0.9, 0.9)))
    cfg.occ_warmup_steps = 8
    cfg.occ_update_interval = 4
    cfg.occ_threshold_scale = 2.5  # a mixed bitfield
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)  # prefetches the warm-up update of step 4 from a fresh stream
    ctx.set_appearance(app.astype(np.float32))
    src = RefRun(cfg, app)
    inject(cfg, None, [src], occupancy_fraction=0.7, table_scale=0.5)
    for g in range(2):
        m, v, _, _ = src.adam(g)
        src.set_adam(g, m, v, 10, 10)  # a state saved at step 10 > occ_warmup_steps
    ref = RefRun(cfg, app)  # fresh Worker + load_state, as a resumed reference run
    with tempfile.TemporaryDirectory() as td:
        for g in range(2):
            path = os.path.join(td, f"s{g}.dgcw")
            src.save_checkpoint(g, HASH, path)
            ctx.load_checkpoint(g, path)
            ref.load_checkpoint(g, path)
    assert ctx.get_step() == 10
    for step in (10, 11):  # the update after step 11 samples 1/4 uniform + 1/4 occupied cells
        o, d, gt, img = workloads.make_rays(cfg, 512, "random", seed=step)
        ctx.train_step(o, d, gt, img, step=step)
        ref.train_step(o, d, gt, img, step)
    for g in range(2):
        for c, box in enumerate(layout.region_boxes(cfg, g)):
            n = int(np.prod(layout.occupancy_shape(cfg, box)))
            dg_den, _ = ctx.occupancy_density(g, c)
            rf_den = ref.occupancy_density(g, c, n)
            close = np.abs(dg_den - rf_den) <= 1e-3 * np.abs(rf_den) + 1e-6
            # a different stream would decay and refresh different cells (~40 % of them)
            assert close.mean() > 0.995, (g, c, close.mean())
            assert np.mean(ctx.get_occupancy(g, c) == ref.occupancy(g, c, n)) > 0.995
