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
