"""GPU: the C++ facade (include/distgrid_b200/distgrid.hpp) used like the reference API —
compiled with g++ against the header, linked to libdg_b200.so, checked against the oracle
(with the reference's own mt19937_64 initialisation on both sides)."""
import os
import subprocess

import numpy as np
import pytest

from oracle.bindings import OracleRun, RefRun, ref_available
from paper_2405_04416_b200 import dg, workloads

from .helpers import small_cfg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_train_and_render(tmp_path):
    exe = tmp_path / "facade_demo"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp"), "-o", str(exe),
                    "-L", os.path.dirname(dg.LIB_PATH), "-ldg_b200",
                    "-Wl,-rpath," + os.path.dirname(dg.LIB_PATH)], check=True)
    cfg = small_cfg(2, 1, table_log2=12, levels=8, nmax=128, divisor=64)
    o, d, gt, _ = workloads.make_rays(cfg, 300, "independent", seed=4)
    gt = gt.astype(np.float32)
    rays = tmp_path / "rays.bin"
    with open(rays, "wb") as f:
        f.write(np.uint64(len(o)).tobytes())
        f.write(np.concatenate([o, d, gt.astype(np.float64)], axis=1).tobytes())
    out = tmp_path / "out.txt"
    subprocess.run([str(exe), str(rays), str(out)], check=True, timeout=300)
    lines = open(out).read().split("\n")
    # oracle with the reference's own init (the facade calls dg_init_params_reference)
    app = np.full((1, 16), 0.25)
    ctx = dg.Context(cfg, device=0)
    orc = OracleRun(cfg, app)
    for g in range(2):
        ctx.init_reference(g)
        orc.set_params(g, ctx.get_params(g).astype(np.float64))
    img = np.zeros(len(o), np.uint32)
    for step in range(2):
        st = orc.train_step(o, d, gt.astype(np.float64), img, step)
        parts = lines[step].split()
        got = [float(x) for x in parts[2:5]]
        want = [st["loss_rgb"], st["loss_transmittance"], st["loss_distortion"]]
        for a, b in zip(got, want):
            assert abs(a - b) <= (1e-4 if step == 0 else 2e-2) * abs(b), (step, a, b)
    rgb, T, depth = orc.eval_rays(o, d, app[0])
    vals = np.array([[float(x) for x in l.split()[1:]] for l in lines if l.startswith("ray ")])
    # after two Adam steps the states drift apart slightly (fp32 vs fp64); renders stay close
    assert np.allclose(vals[:, :3], rgb, rtol=2e-2, atol=2e-3)
    assert "logic_error ok" in lines
    wl = [l for l in lines if l.startswith("workers ")]
    assert wl and wl[0].split() == ["workers", "2", "step", "2", "2", "bytes", "0", "0", "0"], wl
    fl = [l for l in lines if l.startswith("fine_field ")]
    assert fl and fl[0].split() == ["fine_field", "levels", "8", "density_in", "16", "color_in", "47",
                                    "region", "1"], fl
    img_line = [l for l in lines if l.startswith("image ")]
    assert img_line and img_line[0].split()[1:3] == ["16", "12"], img_line
    csum, asum = (float(x) for x in img_line[0].split()[3:5])
    assert np.isfinite(csum) and csum > 0 and np.isfinite(asum), img_line
    if ref_available():
        ref = RefRun(cfg, app)
        for g in range(2):  # reference-exact init, rounded to fp32
            assert np.array_equal(ref.params(g).astype(np.float32), ctx.get_params(g))


def _build(tmp_path, src):
    exe = tmp_path / os.path.splitext(os.path.basename(src))[0]
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, src),
                    "-o", str(exe), "-L", os.path.dirname(dg.LIB_PATH), "-l:libdg_b200.so",
                    "-Wl,-rpath," + os.path.dirname(dg.LIB_PATH)], check=True)
    return exe


def test_cpp_facade_stage_api(tmp_path):
    """The facade's per-function API (include/distgrid/*.hpp: HashGrid, FieldParams,
    query_density / query_color / field_backward per sample and batched, losses, LrSchedule,
    AdamState, segment_ray) against the fp64 oracle.  Bars as the parity suite's stage tests:
    features 1e-5, field outputs 1e-4, field gradients 2e-3 rel-L2 (tcgen05 backward), fp64
    stages (losses, Adam, lr) 1e-12, segments bit-exact."""
    from oracle.bindings import OracleModel
    from .helpers import rel_l2
    exe = _build(tmp_path, "tests/cpp/facade_stages.cpp")
    out = tmp_path / "stages.bin"
    subprocess.run([str(exe), str(out)], check=True, timeout=300)
    v = np.fromfile(out, dtype=np.float64)
    pos = [0]

    def take(n):
        a = v[pos[0]:pos[0] + n]
        pos[0] += n
        return a

    N = 64
    cfg = small_cfg(1, 1, table_log2=12, levels=8, nmax=128)
    ctx = dg.Context(cfg, device=0)
    arrays = ctx.param_layout(0)
    fine = [a for a in arrays if a["cascade"] == 0]
    nf = sum(a["size"] for a in fine)
    ntot = ctx.param_count(0)
    pts = take(3 * N).reshape(N, 3)
    dirs = take(3 * N).reshape(N, 3).astype(np.float32).astype(np.float64)
    app = take(16 * N).reshape(N, 16).astype(np.float32).astype(np.float64)
    pf = take(nf).astype(np.float32).astype(np.float64)  # the device holds fp32 parameters
    params = np.concatenate([pf, np.zeros(ntot - nf)])
    om = OracleModel(cfg)
    enc = take(N * 16).reshape(N, 16)
    enc_ref, _ = om.encode(0, 0, params, pts)
    assert np.allclose(enc, enc_ref, rtol=1e-5, atol=1e-6), np.abs(enc - enc_ref).max()
    dens = take(N * 19).reshape(N, 19)  # sigma, 15 features, rgb
    so, co = om.field_forward(0, 0, params, pts, dirs, app)
    assert np.allclose(dens[:, 0], so, rtol=1e-4, atol=1e-7), np.abs(dens[:, 0] / so - 1).max()
    assert np.allclose(dens[:, 16:19], co, rtol=1e-4, atol=1e-7), np.abs(dens[:, 16:19] - co).max()
    sg = take(N)
    cg = take(3 * N).reshape(N, 3)
    grads = take(nf)
    go = om.field_backward(0, 0, params, pts, dirs, app, sg.astype(np.float32).astype(np.float64),
                           cg.astype(np.float32).astype(np.float64))
    for a in fine:
        s = slice(a["offset"], a["offset"] + a["size"])
        if np.abs(go[s]).max() == 0:
            assert np.abs(grads[s]).max() == 0
            continue
        assert rel_l2(grads[s], go[s]) < 2e-3, (a, rel_l2(grads[s], go[s]))
    # losses (train.cpp:8-75), fp64 kernels
    ab = take(48).reshape(8, 2, 3)
    ra, rb = ab[:, 0], ab[:, 1]
    assert abs(take(1)[0] - np.sum((ra - rb) ** 2)) <= 1e-12 * np.sum((ra - rb) ** 2)
    assert np.allclose(take(3), 2.0 * (ra[0] - rb[0]), rtol=1e-15, atol=0)
    T = take(4)
    tc = np.minimum(T, 1.0 - 1e-6)
    assert abs(take(1)[0] - np.sum(-np.log(1.0 - tc))) <= 1e-12 * np.sum(-np.log(1.0 - tc))
    assert np.allclose(take(4), 1.0 / (1.0 - tc), rtol=1e-15, atol=0)
    w, s_, ds = take(10), take(10), take(10)
    dist = sum(w[i] * w[j] * abs(s_[i] - s_[j]) for i in range(10) for j in range(10)) + np.sum(w * w * ds) / 3
    assert abs(take(1)[0] - dist) <= 1e-12 * dist
    fd = []
    for k in range(10):  # d loss / d w_k of the double sum + interval term
        fd.append(2 * sum(w[j] * abs(s_[k] - s_[j]) for j in range(10)) + 2.0 / 3.0 * w[k] * ds[k])
    assert np.allclose(take(10), fd, rtol=1e-12, atol=1e-15)
    lrs = take(5)
    for st, lr in zip((0, 1, 500, 999, 1000), lrs):
        assert abs(lr - (0.005 + 0.5 * 0.045 * (1 + np.cos(np.pi * st / 1000)))) <= 1e-15
    p0, g1, g2 = take(5), take(5), take(5)
    m = np.zeros(5)
    vv = np.zeros(5)
    p = p0.copy()
    for t, g in ((1, g1), (2, g2)):  # AdamState::step (train.cpp:91-115)
        m = 0.9 * m + (1 - 0.9) * g
        vv = 0.99 * vv + (1 - 0.99) * g * g
        p = p - 0.01 * (m / (1 - 0.9 ** t)) / (np.sqrt(vv / (1 - 0.99 ** t)) + 1e-15)
    assert np.allclose(take(5), p, rtol=1e-14, atol=1e-16)
    assert np.allclose(take(5), m, rtol=1e-14, atol=0) and np.allclose(take(5), vv, rtol=1e-14, atol=0)
    assert take(1)[0] == 2
    # segment_ray, bit-exact against the oracle's restatement (2 x 2 split of a sub-box)
    mc = small_cfg(2, 2, inner=((0.3, 0.25, 0.0), (1.6, 1.8, 0.8)), extent=(2.0, 2.0, 1.0))
    om2 = OracleModel(mc)
    for i in range(32):
        o, d = take(3), take(3)
        ns = int(take(1)[0])
        segs = take(12).reshape(4, 3)
        nseg, region, te, tx = om2.segment_rays(o[None], d[None])
        assert ns == nseg[0], (i, ns, nseg[0])
        for k in range(ns):
            assert segs[k, 0] == region[0, k] and segs[k, 1] == te[0, k] and segs[k, 2] == tx[0, k], (i, k)
    assert pos[0] == len(v)


@pytest.mark.parametrize("name,cases", [("render", 16), ("train", 12)])
def test_reference_unit_tests_on_facade(name, cases):
    """The reference's own unit-test files, compiled UNMODIFIED against the facade headers
    (include/distgrid/) with a doctest-compatible shim by __graft_entry__.build()
    (tests/cpp/Makefile; the reference sources exist only in the build container), run on the
    GPU; every case must pass:
      * test_render.cpp (16 cases): ray_aabb_intersect, march_segment, local_render,
        merge_forward / merge_backward, local_render_backward — golden values and
        finite-difference checks down to 1e-12 (the fp64 stage kernels);
      * test_train.cpp (12 cases): losses and their gradients, the lr schedule, Adam's two-step
        recurrence and shape errors, and the ray cache (refresh ring order, chi-square pixel
        coverage over 1e6 entries, concurrent refresh / draw) on the device ray cache."""
    exe = os.path.join(ROOT, "tests", "cpp", "_build", f"ref_test_{name}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} was not built (reference tree absent at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    summary = [l for l in r.stdout.splitlines() if l.startswith("[doctest] test cases")]
    assert r.returncode == 0 and summary, (r.stdout[-3000:], r.stderr[-3000:])
    assert "| 0 failed" in summary[0] and f"{cases} passed" in summary[0], summary
