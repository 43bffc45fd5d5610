"""Compositing stage entry points of the C ABI (local_render, merge_forward,
merge_backward, local_render_backward, losses) against the oracle's restatements
(oracle/dg_oracle.c or_local_render / or_merge_* / or_loss_* / or_local_render_backward,
render.cpp:46-179, train.cpp:8-75), which the composed-step tests pin bitwise to the reference.
The device computes in fp64 like the reference; outputs round once to fp32, hence the 1e-5 bar
(1e-9 for the fp64 loss outputs)."""
import ctypes as C

import numpy as np
import pytest

from oracle.bindings import oracle_lib
from paper_2405_04416_b200 import dg

from .helpers import small_cfg

pytestmark = pytest.mark.gpu

D = C.POINTER(C.c_double)


def _d(a):
    return np.ascontiguousarray(a, np.float64).ctypes.data_as(D)


def _lib():
    lib = oracle_lib()
    lib.or_local_render.argtypes = [D, D, D, D, C.c_int, D, D, D, D, D]
    lib.or_merge_forward.argtypes = [D, D, D, C.c_int, D, D, D]
    lib.or_merge_backward.argtypes = [D, C.c_double, D, D, C.c_int, D, D]
    lib.or_loss_transmittance.argtypes = [C.c_double, C.c_double]
    lib.or_loss_transmittance.restype = C.c_double
    lib.or_loss_transmittance_grad.argtypes = [C.c_double, C.c_double]
    lib.or_loss_transmittance_grad.restype = C.c_double
    lib.or_loss_distortion.argtypes = [D, D, D, C.c_int]
    lib.or_loss_distortion.restype = C.c_double
    lib.or_loss_distortion_grad.argtypes = [D, D, D, C.c_int, D]
    lib.or_local_render_backward.argtypes = [D, D, D, D, C.c_int, D, C.c_double, D, D, D]
    return lib


def _segments(rng, n_seg, max_len=48):
    lens = rng.integers(0, max_len + 1, n_seg)
    lens[::17] = 0  # empty segments
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    n = int(off[-1])
    t = np.zeros(n)
    delta = rng.uniform(0.005, 0.05, n)
    for g in range(n_seg):
        a, b = int(off[g]), int(off[g + 1])
        t[a:b] = rng.uniform(0.0, 1.0) + np.cumsum(delta[a:b])
    sigma = rng.uniform(0.0, 6.0, n).astype(np.float32)
    sigma[::7] = 0.0
    rgb = rng.uniform(0.0, 1.0, (n, 3)).astype(np.float32)
    return off, t, delta, sigma, rgb


def _close(a, b, rtol=1e-5, atol=1e-7):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.allclose(a, b, rtol=rtol, atol=atol), np.abs(a - b).max()


@pytest.fixture(scope="module")
def ctx():
    return dg.Context(small_cfg(1, 1, table_log2=10, levels=4, nmax=64, divisor=32), device=0)


def test_local_render_and_distortion_stats(ctx):
    lib = _lib()
    rng = np.random.default_rng(5)
    off, t, delta, sigma, rgb = _segments(rng, 300)
    n_seg = len(off) - 1
    t0 = np.array([t[int(off[g])] - 0.01 if off[g + 1] > off[g] else 0.0 for g in range(n_seg)])
    t1 = t0 + rng.uniform(0.5, 3.0, n_seg)
    t1[5] = t0[5]  # zero span: stats stay 0 (render.cpp:83)
    c_rgb, c_T, c_dep, c_dist = ctx.local_render(t, delta, sigma, rgb, off, t0, t1)
    for g in range(n_seg):
        a, b = int(off[g]), int(off[g + 1])
        n = b - a
        orgb, oT, odep = np.zeros(3), np.zeros(1), np.zeros(1)
        alpha, prefix = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        lib.or_local_render(_d(t[a:b]), _d(delta[a:b]), _d(sigma[a:b].astype(np.float64)),
                            _d(rgb[a:b].astype(np.float64).ravel()), n, orgb.ctypes.data_as(D),
                            oT.ctypes.data_as(D), odep.ctypes.data_as(D), alpha.ctypes.data_as(D),
                            prefix.ctypes.data_as(D))
        _close(c_rgb[g], orgb)
        _close(c_T[g], oT[0])
        _close(c_dep[g], odep[0])
        # accumulate_distortion_stats (render.cpp:80-99)
        span = t1[g] - t0[g]
        ws = ms = pair = inter = 0.0
        if span > 0:
            for k in range(n):
                w = prefix[k] * alpha[k]
                s = (t[a + k] - t0[g]) / span
                pair += 2.0 * w * (s * ws - ms)
                inter += w * w * delta[a + k] / span
                ws += w
                ms += w * s
        _close(c_dist[g], [ws, ms, pair + inter / 3.0], rtol=1e-9, atol=1e-12)


def test_local_render_backward(ctx):
    lib = _lib()
    rng = np.random.default_rng(6)
    off, t, delta, sigma, rgb = _segments(rng, 200)
    n_seg, n = len(off) - 1, int(off[-1])
    d_rgb = rng.normal(size=(n_seg, 3)).astype(np.float32)
    d_T = rng.normal(size=n_seg).astype(np.float32)
    w_up = rng.normal(size=n).astype(np.float32)
    for wu in (None, w_up):
        sg, cg = ctx.local_render_backward(t, delta, sigma, rgb, off, d_rgb, d_T, wu)
        for g in range(n_seg):
            a, b = int(off[g]), int(off[g + 1])
            m = b - a
            if m == 0:
                continue
            orgb, oT, odep = np.zeros(3), np.zeros(1), np.zeros(1)
            alpha, prefix = np.zeros(m), np.zeros(m)
            s64, r64 = sigma[a:b].astype(np.float64), rgb[a:b].astype(np.float64).ravel()
            lib.or_local_render(_d(t[a:b]), _d(delta[a:b]), _d(s64), _d(r64), m, orgb.ctypes.data_as(D),
                                oT.ctypes.data_as(D), odep.ctypes.data_as(D), alpha.ctypes.data_as(D),
                                prefix.ctypes.data_as(D))
            osg, ocg = np.zeros(m), np.zeros(3 * m)
            wup = None if wu is None else wu[a:b].astype(np.float64)
            lib.or_local_render_backward(_d(delta[a:b]), _d(r64), alpha.ctypes.data_as(D), prefix.ctypes.data_as(D),
                                         m, _d(d_rgb[g].astype(np.float64)), float(d_T[g]),
                                         None if wup is None else _d(wup), osg.ctypes.data_as(D),
                                         ocg.ctypes.data_as(D))
            _close(sg[a:b], osg, atol=1e-6)
            _close(cg[a:b].ravel(), ocg, atol=1e-7)


def test_merge_forward_backward(ctx):
    lib = _lib()
    rng = np.random.default_rng(7)
    n_rays = 400
    cnt = rng.integers(1, 6, n_rays)
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    ns = int(off[-1])
    srgb = rng.uniform(0, 1, (ns, 3)).astype(np.float32)
    sT = rng.uniform(0, 1, ns).astype(np.float32)
    sT[::11] = 0.0  # opaque segments: no division anywhere
    sdep = rng.uniform(0, 3, ns).astype(np.float32)
    rgb, T, dep = ctx.merge_forward(srgb, sT, sdep, off)
    d_rgb = rng.normal(size=(n_rays, 3)).astype(np.float32)
    d_T = rng.normal(size=n_rays).astype(np.float32)
    g_rgb, g_T = ctx.merge_backward(srgb, sT, off, d_rgb, d_T)
    for r in range(n_rays):
        a, b = int(off[r]), int(off[r + 1])
        m = b - a
        orgb, oT, odep = np.zeros(3), np.zeros(1), np.zeros(1)
        r64, T64, d64 = srgb[a:b].astype(np.float64).ravel(), sT[a:b].astype(np.float64), sdep[a:b].astype(np.float64)
        lib.or_merge_forward(_d(r64), _d(T64), _d(d64), m, orgb.ctypes.data_as(D), oT.ctypes.data_as(D),
                             odep.ctypes.data_as(D))
        _close(rgb[r], orgb)
        _close(T[r], oT[0])
        _close(dep[r], odep[0])
        gc, gt = np.zeros(3 * m), np.zeros(m)
        lib.or_merge_backward(_d(d_rgb[r].astype(np.float64)), float(d_T[r]), _d(r64), _d(T64), m,
                              gc.ctypes.data_as(D), gt.ctypes.data_as(D))
        _close(g_rgb[a:b].ravel(), gc, atol=1e-6)
        _close(g_T[a:b], gt, atol=1e-6)


def test_merge_errors(ctx):
    with pytest.raises(dg.DGError):  # merge: no partials (render.cpp:102)
        ctx.merge_forward(np.zeros((1, 3)), np.ones(1), np.zeros(1), np.array([0, 1, 1], np.uint64))
    with pytest.raises(dg.DGError):  # offsets must start at 0
        ctx.merge_forward(np.zeros((2, 3)), np.ones(2), np.zeros(2), np.array([1, 2], np.uint64))
    with pytest.raises(dg.DGError):  # more partials than any schedule holds
        n = 40
        ctx.merge_backward(np.zeros((n, 3)), np.ones(n), np.array([0, n], np.uint64), np.zeros((1, 3)), np.zeros(1))


def test_losses(ctx):
    lib = _lib()
    rng = np.random.default_rng(8)
    n = 1000
    rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    gt = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    T = rng.uniform(0, 1, n).astype(np.float32)
    T[:5] = 1.0  # the clamp (train.cpp:24-26)
    lr, lt, dr, dt = ctx.ray_losses(rgb, gt, T, eps=1e-6)
    d = rgb.astype(np.float64) - gt.astype(np.float64)
    _close(lr, (d * d).sum(1), rtol=1e-12, atol=0)
    _close(dr, 2.0 * d)
    ot = np.array([lib.or_loss_transmittance(float(x), 1e-6) for x in T])
    og = np.array([lib.or_loss_transmittance_grad(float(x), 1e-6) for x in T])
    _close(lt, ot, rtol=1e-12, atol=0)
    _close(dt, og)
    # distortion
    off, t, delta, sigma, _ = _segments(rng, 150)
    n_seg, m = len(off) - 1, int(off[-1])
    w = rng.uniform(0, 0.2, m)
    s = np.zeros(m)
    ds = rng.uniform(0.001, 0.02, m)
    for g in range(n_seg):
        a, b = int(off[g]), int(off[g + 1])
        s[a:b] = np.sort(rng.uniform(0, 1, b - a))
    loss, grads = ctx.distortion_loss(w, s, ds, off)
    for g in range(n_seg):
        a, b = int(off[g]), int(off[g + 1])
        k = b - a
        ol = lib.or_loss_distortion(_d(w[a:b]), _d(s[a:b]), _d(ds[a:b]), k)
        og = np.zeros(max(k, 1))
        lib.or_loss_distortion_grad(_d(w[a:b]), _d(s[a:b]), _d(ds[a:b]), k, og.ctypes.data_as(D))
        _close(loss[g], ol, rtol=1e-12, atol=1e-15)
        _close(grads[a:b], og[:k], rtol=1e-12, atol=1e-15)
