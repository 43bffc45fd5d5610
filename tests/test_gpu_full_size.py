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
