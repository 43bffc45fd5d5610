"""CPU: known-answer tests from the reference's own unit tests, checked against the oracle
restatement (oracle/dg_oracle.c), plus the committed golden fixture produced by the
reference build (tests/golden/make_golden.py).  These run without /root/reference."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.bindings import OracleModel, OracleRun, oracle_lib
from paper_2405_04416_b200 import layout, workloads
from paper_2405_04416_b200.abi import RunConfig

from .helpers import small_cfg

HERE = os.path.dirname(os.path.abspath(__file__))
P = C.c_void_p
D3 = C.c_double * 3


def lib():
    L = oracle_lib()
    L.or_ray_aabb.argtypes = [P, P, P, P, P]
    L.or_grid_shape.restype = C.c_uint32 * 3
    L.or_merge_forward.argtypes = [P, P, P, C.c_int, P, P, P]
    L.or_merge_backward.argtypes = [P, C.c_double, P, P, C.c_int, P, P]
    L.or_loss_transmittance.restype = C.c_double
    L.or_loss_transmittance.argtypes = [C.c_double, C.c_double]
    L.or_loss_transmittance_grad.restype = C.c_double
    L.or_loss_transmittance_grad.argtypes = [C.c_double, C.c_double]
    L.or_march_segment.argtypes = [C.c_double, C.c_double, P, C.c_int, C.c_double, C.c_int,
                                   C.c_uint64, C.c_uint64, C.c_uint64, P, P, C.c_int]
    L.or_adam_step.argtypes = [P, P, P, P, C.c_uint64, C.c_double, C.c_double, C.c_double,
                               C.c_double, C.c_uint64]
    return L


def ptr(a):
    return a.ctypes.data_as(P)


def test_ray_aabb_axis_aligned():  # test_render.cpp:31-54
    box = np.array([0, 0, 0, 1, 1, 1], dtype=np.float64)
    o = np.array([-1, 0.5, 0.5])
    d = np.array([1.0, 0, 0])
    tn, tf = np.zeros(1), np.zeros(1)
    assert lib().or_ray_aabb(ptr(o), ptr(d), ptr(box), ptr(tn), ptr(tf)) == 1
    assert (tn[0], tf[0]) == (1.0, 2.0)
    o2 = np.array([-1, 2.0, 0.5])
    assert lib().or_ray_aabb(ptr(o2), ptr(d), ptr(box), ptr(tn), ptr(tf)) == 0
    d2 = np.array([-1.0, 0, 0])
    assert lib().or_ray_aabb(ptr(o), ptr(d2), ptr(box), ptr(tn), ptr(tf)) == 0


def test_segment_ray_planar_split():  # test_partition.cpp:204-229
    cfg = small_cfg(2, 1)
    for a, (lo, hi) in enumerate(((-1, 1), (-1, 1), (0, 1))):
        cfg.inner_lo[a] = cfg.outer_lo[a] = lo
        cfg.inner_hi[a] = cfg.outer_hi[a] = hi
    om = OracleModel(cfg)
    ns, reg, te, tx = om.segment_rays(np.array([[-2.0, 0.0, 0.5]]), np.array([[1.0, 0, 0]]))
    assert ns[0] == 2 and list(reg[0, :2]) == [0, 1]
    assert (te[0, 0], tx[0, 0], te[0, 1], tx[0, 1]) == (1.0, 2.0, 2.0, 3.0)
    ns, _, _, _ = om.segment_rays(np.array([[-2.0, 5.0, 0.5]]), np.array([[1.0, 0, 0]]))
    assert ns[0] == 0


def test_march_midpoint_ladder():  # test_render.cpp:80-92
    iv = np.array([0.0, 1.0])
    t, dl = np.zeros(16), np.zeros(16)
    n = lib().or_march_segment(0.0, 1.0, ptr(iv), 1, 0.25, 0, 0, 0, 0, ptr(t), ptr(dl), 16)
    assert n == 4
    assert np.allclose(t[:4], 0.125 + 0.25 * np.arange(4)) and np.all(dl[:4] == 0.25)


def test_grid_shapes_and_levels():  # test_grid.cpp:26-66
    assert layout.grid_shape((2, 1, 1), 8) == (8, 4, 4)
    assert layout.grid_shape((3, 2, 1), 10) == (10, 7, 4)
    assert layout.grid_shape((1, 1, 1), 16) == (16, 16, 16)
    L = oracle_lib()
    assert L.or_level_resolution(8, 16, 512, 0) == 16
    assert L.or_level_resolution(8, 16, 512, 7) == 512
    for l in range(8):
        assert layout.level_resolution(8, 16, 512, l) == L.or_level_resolution(8, 16, 512, l)


def test_table_index_known_answers():  # test_grid.cpp:87-125
    cfg = small_cfg(1, 1, table_log2=19, levels=1, nmax=16)
    cfg.base_resolution = 4
    cfg.max_resolution = 4
    om = OracleModel(cfg)
    p = np.zeros(layout.partition_param_count(cfg, 0))
    pts = np.array([[1 / 3, 2 / 3, 1.0]])  # vertex (1, 2, 3) of a 4^3 lattice
    _, rows = om.encode(0, 0, p, pts)
    assert 57 in rows[0, 0]
    # hashed mode vs an exact-integer oracle
    cfg2 = small_cfg(1, 1, table_log2=19, levels=1, nmax=1024)
    cfg2.base_resolution = cfg2.max_resolution = 1024
    om2 = OracleModel(cfg2)
    rng = np.random.default_rng(11)
    p2 = np.zeros(layout.partition_param_count(cfg2, 0))
    for _ in range(50):
        v = rng.integers(0, 1023, 3)
        pt = (v / 1023.0)[None, :]
        _, rows = om2.encode(0, 0, p2, pt)
        want = (int(v[0]) ^ (int(v[1]) * 2654435761) ^ (int(v[2]) * 805459861)) % (1 << 19)
        assert want in rows[0, 0]


def test_merge_worked_example_and_backward():  # test_render.cpp:197-256
    L = lib()
    rgb = np.array([[0.2] * 3, [0.4] * 3, [0.8] * 3])
    T = np.array([0.5, 0.5, 0.5])
    c, t, dep = np.zeros(3), np.zeros(1), np.zeros(1)
    L.or_merge_forward(ptr(rgb), ptr(T), None, 3, ptr(c), ptr(t), ptr(dep))
    assert abs(c[0] - 0.6) < 1e-15 and abs(t[0] - 0.125) < 1e-15
    rgb2 = np.array([[0.2] * 3, [0.4] * 3])
    T2 = np.array([0.5, 0.8])
    up = np.array([1.0, 0, 0])
    gc, gt = np.zeros(6), np.zeros(2)
    L.or_merge_backward(ptr(up), 0.0, ptr(rgb2), ptr(T2), 2, ptr(gc), ptr(gt))
    assert (gc[0], gc[3]) == (1.0, 0.5)
    assert abs(gt[0] - 0.4) < 1e-15 and gt[1] == 0.0


def test_losses_and_lr():  # test_train.cpp:11-99
    L = lib()
    assert L.or_loss_transmittance(0.0, 1e-6) == 0.0
    assert abs(L.or_loss_transmittance_grad(0.5, 1e-6) - 2.0) < 1e-15
    assert abs(L.or_loss_transmittance(1.0, 1e-6) + np.log(1e-6)) < 1e-9
    cfg = RunConfig()
    cfg.lr_start, cfg.lr_end, cfg.total_steps = 0.05, 0.005, 1000
    assert abs(oracle_lib().or_lr_at(C.byref(cfg), 0) - 0.05) < 1e-15
    assert abs(oracle_lib().or_lr_at(C.byref(cfg), 1000) - 0.005) < 1e-15


def test_adam_two_step_recurrence():  # test_train.cpp:122-152
    L = lib()
    p = np.array([0.7])
    m, v = np.zeros(1), np.zeros(1)
    g1, g2, lr = 0.3, -0.1, 0.01
    mm = 0.1 * g1
    vv = 0.01 * g1 * g1
    want = 0.7 - lr * (mm / 0.1) / (np.sqrt(vv / 0.01) + 1e-15)
    mm = 0.9 * mm + 0.1 * g2
    vv = 0.99 * vv + 0.01 * g2 * g2
    want -= lr * (mm / (1 - 0.81)) / (np.sqrt(vv / (1 - 0.99 * 0.99)) + 1e-15)
    for t, g in ((1, g1), (2, g2)):
        gg = np.array([g])
        L.or_adam_step(ptr(p), ptr(gg), ptr(m), ptr(v), 1, lr, 0.9, 0.99, 1e-15, t)
    assert abs(p[0] - want) < 1e-14


def test_zero_field_gives_unit_sigma_and_grey():  # test_field.cpp:85-100
    cfg = small_cfg(1, 1, table_log2=8, levels=3, nmax=16)
    om = OracleModel(cfg)
    p = np.zeros(layout.partition_param_count(cfg, 0))
    s, c = om.field_forward(0, 0, p, np.array([[0.5, 0.5, 0.5]]), np.array([[0, 0, 1.0]]),
                            np.zeros((1, 16)))
    assert s[0] == 1.0 and np.all(c == 0.5)


def test_golden_fixture_from_reference_build():
    path = os.path.join(HERE, "golden", "golden_small.npz")
    z = np.load(path)
    cfg = RunConfig.from_buffer_copy(z["cfg"].tobytes())
    app = z["app"]
    orc = OracleRun(cfg, app)
    P = cfg.kx * cfg.ky
    for g in range(P):
        orc.set_params(g, z[f"params0_{g}"])
    for c, name in enumerate(("occ_fine", "occ_coarse")):
        for g in range(P):
            orc.set_occupancy(g, c, z[f"{name}_{g}"])
    st = orc.train_step(z["o"], z["d"], z["gt"], z["img"], int(z["step"]))
    assert np.array_equal(np.array([st["loss_rgb"], st["loss_transmittance"], st["loss_distortion"]]),
                          z["losses"])
    for g in range(P):
        assert np.array_equal(orc.params(g), z[f"params1_{g}"])
    rgb, T, depth = orc.eval_rays(z["o"], z["d"], app[0])
    assert np.array_equal(rgb, z["eval_rgb"]) and np.array_equal(T, z["eval_T"])
    assert np.array_equal(depth, z["eval_depth"])
    nseg, reg, te, tx = OracleModel(cfg).segment_rays(z["o"], z["d"])
    assert np.array_equal(nseg, z["nseg"]) and np.array_equal(te, z["te"])
