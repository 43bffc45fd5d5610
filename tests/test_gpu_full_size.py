"""Full-size properties (BASELINE C4 weak point, the bench workload: T = 2^24, L = 16,
Nmax = 2048, 131,072 drift rays on one partition), where the fp64 oracle cannot run the whole
step: on random subsets, everything the index path produces is the reference's bit for bit —
segments, the items each partition receives (in ray order), per-item sample counts and
t / delta of a training step, and the hash-table rows of the encoded samples — and the step's
outputs are finite and reproducible."""
import numpy as np
import pytest

from oracle.bindings import OracleModel
from paper_2405_04416_b200 import dg, layout, workloads

pytestmark = pytest.mark.gpu


def test_full_size_index_path_bit_exact():
    wl = workloads.weak(1)
    cfg = wl.cfg
    ctx = dg.Context(cfg, device=0)
    ctx.init_fast(0, seed=1)
    ctx.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))
    o, d, gt, img = workloads.make_rays(cfg, wl.n_rays, wl.generator, seed=1)
    st = ctx.train_step(o, d, gt, img, step=0)
    assert all(np.isfinite(st[k]) for k in ("loss_rgb", "loss_transmittance", "loss_distortion"))
    assert st["rays"] == wl.n_rays
    om = OracleModel(cfg)
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(wl.n_rays, 1500, replace=False))
    # segments
    ns_g, reg_g, te_g, tx_g = ctx.segment_rays(o[pick], d[pick])
    ns_o, reg_o, te_o, tx_o = om.segment_rays(o[pick], d[pick])
    assert np.array_equal(ns_g, ns_o)
    m = np.arange(16)[None, :] < ns_o[:, None]
    assert np.array_equal(np.where(m, te_g, 0).view(np.uint64), np.where(m, te_o, 0).view(np.uint64))
    assert np.array_equal(np.where(m, tx_g, 0).view(np.uint64), np.where(m, tx_o, 0).view(np.uint64))
    # items of the step: every intersecting ray, in ray order
    rid, order, te, tx, cnt = ctx.last_item_data(0)
    assert np.all(np.diff(rid.astype(np.int64)) > 0)
    # march of a subset of items: counts, t, delta bit-exact (jitter on, batch 0)
    t_g, dl_g, c_g = ctx.last_samples(0)
    off = np.concatenate([[0], np.cumsum(cnt.astype(np.int64))])
    sub = np.sort(rng.choice(len(rid), 400, replace=False))
    occ = [np.ones(int(np.prod(layout.occupancy_shape(cfg, b))), np.uint8) for b in layout.region_boxes(cfg, 0)]
    r = rid[sub].astype(np.int64)
    # benchmark mode (wire_f32): the owner marches the f32-rounded dispatch payload
    # (WireWriter::real, wire.hpp:55-62), as the reference worker does
    ow, dw = (o[r].astype(np.float32).astype(np.float64), d[r].astype(np.float32).astype(np.float64)) \
        if cfg.wire_f32 else (o[r], d[r])
    co, to, do, _ = om.cascade_march(0, occ[0], occ[1], ow, dw, te[sub], tx[sub], rid[sub], 1, 0)
    assert np.array_equal(cnt[sub], co)
    want_t = np.concatenate([t_g[off[i]:off[i + 1]] for i in sub])
    want_d = np.concatenate([dl_g[off[i]:off[i + 1]] for i in sub])
    assert np.array_equal(want_t.view(np.uint64), to.view(np.uint64))
    assert np.array_equal(want_d.view(np.uint64), do.view(np.uint64))
    # hash-table rows of encoded sample positions (all 16 levels, hashed and one-to-one)
    fine, _ = layout.region_boxes(cfg, 0)
    lo, hi = np.array(fine[0]), np.array(fine[1])
    ii = sub[:200]
    pts = []
    for i in ii:
        k = int(rid[i])
        ts = t_g[off[i]:off[i + 1]][:8]
        ok, dk = (o[k].astype(np.float32).astype(np.float64), d[k].astype(np.float32).astype(np.float64)) \
            if cfg.wire_f32 else (o[k], d[k])
        p = (ok[None, :] + dk[None, :] * ts[:, None] - lo) / (hi - lo)
        pts.append(np.clip(p, 0.0, 1.0))
    pts = np.concatenate(pts)
    _, rows_g = ctx.encode(0, 0, pts)
    rows_o = om.encode_rows(0, 0, pts)
    assert np.array_equal(rows_g, rows_o)
    assert (rows_o[:, 15, :] != 0xffffffff).any()
    # reproducible: the same batch again from the same state gives the same losses
    ctx2 = dg.Context(cfg, device=0)
    ctx2.init_fast(0, seed=1)
    ctx2.set_appearance(workloads.appearance_rows(cfg.appearance_dim, 1))
    st2 = ctx2.train_step(o, d, gt, img, step=0)
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(st2[k] - st[k]) <= 1e-9 * abs(st[k]), k


# ------------------------------------------------------------------ value parity at the bench config
def _full_pair(wl, table_scale=0.5):
    """GPU context + oracle run of a whole workload config from identical injected fp32 state."""
    from oracle.bindings import OracleRun

    from .helpers import app_rows, inject
    cfg = wl.cfg
    app = app_rows(1)
    ctx = dg.Context(cfg, device=0)
    ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    inject(cfg, ctx, [orc], table_scale=table_scale)
    return ctx, orc


def _grad_parity(cfg, ctx, orc, p0, lr, tol=1e-4):
    from .helpers import rel_l2
    for g in range(cfg.kx * cfg.ky):
        m_g, _, _ = ctx.get_adam(g)
        grad_g = m_g.astype(np.float64) / (1.0 - cfg.adam_beta1)  # first Adam step from m = 0
        grad_o = orc.grads(g)
        worst = 0.0
        for arr in ctx.param_layout(g):
            a = slice(arr["offset"], arr["offset"] + arr["size"])
            if np.abs(grad_o[a]).max() == 0:
                assert np.abs(grad_g[a]).max() < 1e-20, arr
                continue
            e = rel_l2(grad_g[a], grad_o[a])
            worst = max(worst, e)
            assert e < tol, (arr, e)
        big = np.abs(grad_o) > 1e-6 * np.abs(grad_o).max()
        err = np.abs((ctx.get_params(g).astype(np.float64) - p0[g]) - (orc.params(g) - p0[g]))
        assert np.mean(err[big] <= 1e-3 * lr) >= 0.999, np.mean(err[big] <= 1e-3 * lr)
        print("worst per-array gradient rel-L2", worst)


@pytest.mark.slow
def test_full_size_value_parity_c4_weak_1():
    """The benchmarked configuration exactly (C4-weak-1: T = 2^24, L = 16, Nmax = 2048, march
    divisor 104, wire_f32 = 1, default encode pass budgets, so the backward cuts every hashed
    level into S = 2 row slices) on a 2,048-ray subset of the bench batch, against the fp64
    oracle from identical injected state: losses and render within 1e-4, per-array gradients
    (relative L2) within 1e-4, Adam within 1e-3 lr on 99.9 % of the entries, sample positions
    and encoded features through dg_last_sample_data."""
    from .helpers import params_for, tied_train_step
    wl = workloads.weak(1)
    cfg = wl.cfg
    assert cfg.fine_table_log2 == 24 and cfg.max_resolution == 2048 and cfg.wire_f32 == 1
    assert cfg.march_step_divisor == 104.0
    ctx, orc = _full_pair(wl)
    o, d, gt, img = workloads.make_rays(cfg, wl.n_rays, wl.generator, seed=1)
    pick = np.sort(np.random.default_rng(5).choice(wl.n_rays, 2048, replace=False))
    o, d, gt, img = o[pick], d[pick], gt[pick], img[pick]
    # render first (identical state on both sides)
    app = np.asarray(orc.app[0])
    rgb, T, depth = ctx.render(o, d, app)
    rgb_o, T_o, depth_o = orc.eval_rays(o, d, app)
    assert np.allclose(rgb, rgb_o, rtol=1e-4, atol=1e-6), np.abs(rgb - rgb_o).max()
    assert np.allclose(T, T_o, rtol=1e-4, atol=1e-6), np.abs(T - T_o).max()
    assert np.allclose(depth, depth_o, rtol=1e-4, atol=1e-5), np.abs(depth - depth_o).max()
    p0 = [params_for(cfg, 0, table_scale=0.5).astype(np.float64)]
    orc.log_samples(0, 400_000)
    sg, so, (ties, zmax) = tied_train_step(ctx, orc, o, d, gt, img, 0)
    assert ties <= 64 and zmax <= 4e-6, (ties, zmax)
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(sg[k] - so[k]) <= 1e-4 * abs(so[k]), (k, sg[k], so[k])
    pos, x, out, up, dx = ctx.last_sample_data(0)
    pos_o, x_o, out_o, up_o, dx_o = orc.sample_log()
    assert len(pos) == len(pos_o) > 100_000
    assert np.array_equal(pos.view(np.uint64), pos_o.view(np.uint64))
    assert (np.abs(x - x_o) / np.maximum(np.abs(x_o).max(axis=0), 1e-30)).max() < 1e-5
    assert (np.abs(out - out_o) / np.maximum(np.abs(out_o), 1e-6)).max() < 1e-5
    _grad_parity(cfg, ctx, orc, p0, sg["lr"])


@pytest.mark.parametrize("mb", [None, 1])
def test_value_parity_c1_grid(mb, monkeypatch):
    """C1's grid (T = 2^19, L = 16, Nmax = 2048, vertical rays, divisor 128) on 2,048 rays; with
    mb = 1 the encode passes are cut to 1 MB row slices (4 per hashed level), so the
    forward's k > 0 slices add into the features and the backward's clip_to_slice runs."""
    from .helpers import params_for, tied_train_step
    if mb is not None:
        monkeypatch.setenv("DG_ENC_FWD_MB", str(mb))
        monkeypatch.setenv("DG_ENC_BWD_MB", str(mb))
    wl = workloads.c1()
    cfg = wl.cfg
    ctx, orc = _full_pair(wl)
    o, d, gt, img = workloads.make_rays(cfg, 2048, wl.generator, seed=3)
    p0 = [params_for(cfg, 0, table_scale=0.5).astype(np.float64)]
    sg, so, (ties, zmax) = tied_train_step(ctx, orc, o, d, gt, img, 0)
    assert ties <= 64 and zmax <= 4e-6, (ties, zmax)
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(sg[k] - so[k]) <= 1e-4 * abs(so[k]), (k, sg[k], so[k])
    _grad_parity(cfg, ctx, orc, p0, sg["lr"])


@pytest.mark.slow
def test_value_parity_c2_two_partitions_on_one_gpu():
    """C2's configuration (2 x 1 partitions, T = 2^22 per partition, Nmax = 2048, divisor 193,
    independent rays: ~50 % cross the plane) with both partitions on one GPU, on a 2,048-ray
    subset: per-field encode passes over two fields' hashed and paired one-to-one tables, the
    sample order per field, the aliased partial exchange and two-segment merges, against the
    fp64 oracle from identical injected state (render, losses, per-array gradients, Adam)."""
    from .helpers import params_for, tied_train_step
    wl = workloads.c2()
    cfg = wl.cfg
    assert cfg.kx == 2 and cfg.fine_table_log2 == 22
    ctx, orc = _full_pair(wl)
    o, d, gt, img = workloads.make_rays(cfg, 2048, wl.generator, seed=11)
    app = np.asarray(orc.app[0])
    rgb, T, depth = ctx.render(o, d, app)
    rgb_o, T_o, depth_o = orc.eval_rays(o, d, app)
    assert np.allclose(rgb, rgb_o, rtol=1e-4, atol=1e-6), np.abs(rgb - rgb_o).max()
    assert np.allclose(T, T_o, rtol=1e-4, atol=1e-6), np.abs(T - T_o).max()
    p0 = [params_for(cfg, g, table_scale=0.5).astype(np.float64) for g in range(2)]
    sg, so, (ties, zmax) = tied_train_step(ctx, orc, o, d, gt, img, 0)
    assert ties <= 64 and zmax <= 4e-6, (ties, zmax)
    assert sg["rays"] == so["rays"] == 2048
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(sg[k] - so[k]) <= 1e-4 * abs(so[k]), (k, sg[k], so[k])
    _grad_parity(cfg, ctx, orc, p0, sg["lr"])
