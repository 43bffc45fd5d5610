"""CPU: pin the C restatement (oracle/dg_oracle.c) to the reference library itself.

The reference (oracle/_ref/libdistgrid_ref.so) is the unmodified /root/reference build; both
are fp64 with contraction off, so agreement is bit for bit: segments, samples, encodings,
composed train steps (losses, every parameter after Adam, Adam moments), occupancy updates,
evaluation renders, and the wire_f32 rounding semantics.
"""
import numpy as np
import pytest

from oracle.bindings import OracleModel, OracleRun, RefRun, ref_available, ref_segment_rays
from paper_2405_04416_b200 import layout, workloads

from .helpers import app_rows, inject, params_for, small_cfg

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def same(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("kx,ky,gen", [(1, 1, "vertical"), (2, 1, "independent"),
                                       (2, 2, "random"), (4, 2, "corner"), (5, 3, "random")])
def test_segments_identical(kx, ky, gen):
    cfg = small_cfg(kx, ky)
    o, d, _, _ = workloads.make_rays(cfg, 3000, gen, seed=2)
    d[:3] = [[0, 0, -1.0], [1.0, 0, 0], [0, 1.0, 0]]
    r = ref_segment_rays(cfg, o, d)
    m = OracleModel(cfg).segment_rays(o, d)
    for a, b in zip(r, m):
        assert same(a, b)


@pytest.mark.parametrize("jitter", [0, 1])
def test_cascade_march_identical(jitter):
    cfg = small_cfg(2, 1, inner=((0.4, 0.2, 0.0), (1.5, 0.9, 0.8)), occ_res=20)
    ref = RefRun(cfg, app_rows())
    om = OracleModel(cfg)
    o, d, _, _ = workloads.make_rays(cfg, 600, "random", seed=4)
    ns, reg, te, tx = om.segment_rays(o, d)
    rng = np.random.default_rng(3)
    for g in range(2):
        occ = []
        for c, box in enumerate(layout.region_boxes(cfg, g)):
            sh = layout.occupancy_shape(cfg, box)
            bits = (rng.random(sh[0] * sh[1] * sh[2]) < 0.6).astype(np.uint8)
            ref.set_occupancy(g, c, bits)
            occ.append(bits)
        sel = [(i, s) for i in range(len(o)) for s in range(ns[i]) if reg[i, s] == g]
        idx = np.array([i for i, _ in sel])
        t0 = np.array([te[i, s] for i, s in sel])
        t1 = np.array([tx[i, s] for i, s in sel])
        rid = idx.astype(np.uint64)
        a = ref.cascade_march(g, o[idx], d[idx], t0, t1, rid, jitter, 9)
        b = om.cascade_march(g, occ[0], occ[1], o[idx], d[idx], t0, t1, rid, jitter, 9)
        for x, y in zip(a, b):
            assert same(x, y)


def test_encode_and_field_identical():
    cfg = small_cfg(1, 1, table_log2=12, levels=8, nmax=256, extent=(1.3, 1.0, 0.7))
    ref = RefRun(cfg, app_rows())
    om = OracleModel(cfg)
    p = params_for(cfg, 0, table_scale=0.5)
    ref.set_params(0, p)
    rng = np.random.default_rng(5)
    pts = rng.random((300, 3))
    dirs = rng.normal(size=(300, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    app = rng.uniform(-1, 1, (300, 16))
    for c in (0, 1):
        e1, r1 = ref.encode(0, c, pts)
        e2, r2 = om.encode(0, c, p, pts)
        assert same(e1, e2) and same(r1, r2)
        s1, c1 = ref.field_forward(0, c, pts, dirs, app)
        s2, c2 = om.field_forward(0, c, p, pts, dirs, app)
        assert same(s1, s2) and same(c1, c2)
        ds = rng.uniform(-1, 1, 300)
        dr = rng.uniform(-1, 1, (300, 3))
        ref.field_backward(0, c, pts, dirs, app, ds, dr)
        g1 = ref.stage_grads(0, zero=True)
        g2 = om.field_backward(0, c, p, pts, dirs, app, ds, dr)
        assert same(g1, g2)


@pytest.mark.parametrize("kx,ky,wire_f32,occ", [(1, 1, 0, None), (2, 1, 0, None), (2, 2, 1, 0.7),
                                                (3, 2, 0, 0.5)])
def test_train_and_eval_identical(kx, ky, wire_f32, occ):
    inner = ((0.2, 0.1, 0.0), (kx - 0.3, ky - 0.2, 0.9)) if occ else None
    cfg = small_cfg(kx, ky, table_log2=12, levels=6, nmax=128, divisor=48, inner=inner,
                    wire_f32=wire_f32, occ_res=16)
    app = app_rows(2)
    ref, orc = RefRun(cfg, app), OracleRun(cfg, app)
    inject(cfg, None, [ref, orc], occupancy_fraction=occ)
    o, d, gt, img = workloads.make_rays(cfg, 300, "random", seed=kx * ky)
    img[::2] = 1
    for step in (14, 15, 16):  # crosses an occupancy update (step_ % 16 == 0)
        s1 = ref.train_step(o, d, gt, img, step)
        s2 = orc.train_step(o, d, gt, img, step)
        assert s1 == s2
    for g in range(kx * ky):
        assert same(ref.params(g), orc.params(g))
        m1, v1, t1, w1 = ref.adam(g)
        m2, v2, t2, w2 = orc.adam(g)
        assert same(m1, m2) and same(v1, v2) and t1 == t2 and w1 == w2
        for c, box in enumerate(layout.region_boxes(cfg, g)):
            sh = layout.occupancy_shape(cfg, box)
            n = sh[0] * sh[1] * sh[2]
            assert same(ref.occupancy(g, c, n), orc.occupancy(g, c, n))
    a = ref.eval_rays(o, d, app[1])
    b = orc.eval_rays(o, d, app[1])
    for x, y in zip(a, b):
        assert same(x, y)


def _camera_rays(cam):
    """Pixel-centre rays of a camera (row-major) through the oracle's make_pixel_ray, which
    tests/test_ray_cache.py pins bitwise to the reference."""
    import ctypes as C
    from oracle.bindings import oracle_lib
    from paper_2405_04416_b200.abi import cameras
    L = oracle_lib()
    L.or_make_pixel_ray.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]
    k = cameras([cam])
    img = np.zeros((cam["height"], cam["width"], 3), np.uint8)
    n = cam["width"] * cam["height"]
    o, d, col = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(3)
    iid, pid = C.c_uint32(), C.c_uint64()
    for y in range(cam["height"]):
        for x in range(cam["width"]):
            i = y * cam["width"] + x
            L.or_make_pixel_ray(C.cast(k, C.c_void_p), img.ctypes.data, x, y, o[i].ctypes.data, d[i].ctypes.data,
                                col.ctypes.data, C.byref(iid), C.byref(pid))
    return o, d


def eval_camera(kx=2, ky=2):
    """A camera above a kx x ky scene looking down at its centre (rays cross regions)."""
    pos = np.array([kx * 0.5 + 0.3, ky * 0.5 - 0.2, 2.2])
    fwd = np.array([kx * 0.5, ky * 0.5, 0.0]) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 1.0, 0.0])
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return dict(image_id=0, width=24, height=18, is_train=1, rotation=np.stack([right, down, fwd], axis=1),
                translation=pos, fx=14.0, fy=14.5, cx=12.2, cy=8.9)


@pytest.mark.parametrize("early", [0, 1])
def test_eval_image_attribution_and_early_termination(early):
    """evaluate_image (worker.cpp:836-880) with and without the driver's early termination
    (worker.cpp:815-818): the restatement's colour, T, depth and attribution are the
    reference's, bitwise."""
    cfg = small_cfg(2, 2, table_log2=12, levels=6, nmax=128, divisor=48, occ_res=16)
    cfg.eval_early_termination = early
    cfg.eval_termination_threshold = 0.6
    app = app_rows(1)
    ref, orc = RefRun(cfg, app), OracleRun(cfg, app)
    inject(cfg, None, [ref, orc], table_scale=0.5)
    cam = eval_camera()
    o, d = _camera_rays(cam)
    a = ref.eval_image(cam, app[0])
    b = orc.eval_rays_attribution(o, d, app[0])
    for x, y in zip(a, b):
        assert same(x, y)
    assert np.abs(a[3]).sum() > 0
