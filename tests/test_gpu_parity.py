"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical inputs.

Bars (BASELINE.json north_star):
  * ray-segment assignment, sample positions (t, delta, cascade) and hash indices: bit-exact;
  * rendered RGB / T / depth and the three losses: within 1e-4 relative (fp32 path);
  * gradients: relative L2 <= 1e-4 over each parameter array on the default tcgen05 path
    (atomics reorder sums), with the oracle given the GPU's ReLU on/off decisions
    (helpers.tied_train_step): a unit whose fp64 pre-activation lies within fp32 noise of 0
    rounds to either side and switches its whole gradient contribution, so each such tie is
    checked separately -- at most a handful per step, every one with |z| <= 4e-6;
  * Adam: |dp_gpu - dp_ref| <= 1e-3 * lr for >= 99.9 % of the entries with |g| > 1e-6 * max|g|.
The FFMA fp32 path (DG_MLP=ffma) recomputes its masks in the backward and is compared untied
(its bars in TOLS).
"""
import numpy as np
import pytest

from oracle.bindings import OracleModel, OracleRun
from paper_2405_04416_b200 import dg, layout, workloads

from .helpers import app_rows, inject, rel_err, rel_l2, small_cfg, tied_train_step

pytestmark = pytest.mark.gpu

LOSSES = ("loss_rgb", "loss_transmittance", "loss_distortion")


def _rays(cfg, n, gen, seed):
    return workloads.make_rays(cfg, n, gen, seed=seed)


# ------------------------------------------------------------------ stage 1
@pytest.mark.parametrize("kx,ky,gen", [(1, 1, "vertical"), (2, 1, "independent"),
                                       (2, 2, "independent"), (4, 2, "drift"), (4, 2, "corner"),
                                       (3, 5, "random")])
def test_segments_bit_exact(kx, ky, gen):
    cfg = small_cfg(kx, ky)
    o, d, _, _ = _rays(cfg, 4000, gen, seed=kx * 10 + ky)
    # edge cases: axis-aligned directions (d == 0 slab rule), rays starting inside, misses
    o[:8] = [[0.5, 0.5, 2.0]] * 8
    d[:4] = [[0.0, 0.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    d[4:8] = [[-1.0, 0.0, 0.0], [0.6, 0.8, 0.0], [0.0, -0.6, -0.8], [0.0, 0.0, -1.0]]
    o[7] = [kx + 5.0, 0.5, 0.5]  # misses the box
    # rays running exactly on partition planes / plane intersections, and grazing a box face
    o[8:12] = [[1.0, 0.5, 2.0], [1.0, 1.0, 2.0], [0.25, 1.0, 2.0], [0.0, 0.3, 2.0]]
    d[8:12] = [[0.0, 0.0, -1.0]] * 4
    ctx = dg.Context(cfg, device=0)
    ns_g, reg_g, te_g, tx_g = ctx.segment_rays(o, d)
    ns_o, reg_o, te_o, tx_o = OracleModel(cfg).segment_rays(o, d)
    assert np.array_equal(ns_g, ns_o)
    mask = np.arange(16)[None, :] < ns_o[:, None]
    assert np.array_equal(np.where(mask, reg_g, 0), np.where(mask, reg_o, 0))
    assert np.array_equal(np.where(mask, te_g, 0).view(np.uint64), np.where(mask, te_o, 0).view(np.uint64))
    assert np.array_equal(np.where(mask, tx_g, 0).view(np.uint64), np.where(mask, tx_o, 0).view(np.uint64))
    if kx * ky > 1:
        assert (ns_o > 1).any()


# ------------------------------------------------------------------ stage 2
@pytest.mark.parametrize("jitter", [0, 1])
@pytest.mark.parametrize("frac", [1.0, 0.55])
def test_cascade_march_bit_exact(jitter, frac):
    cfg = small_cfg(2, 2, inner=((0.3, 0.2, 0.1), (1.7, 1.8, 0.9)), occ_res=24)
    ctx = dg.Context(cfg, device=0)
    om = OracleModel(cfg)
    o, d, _, _ = _rays(cfg, 1500, "random", seed=5)
    ns, reg, te, tx = om.segment_rays(o, d)
    rng = np.random.default_rng(1)
    for g in range(4):
        fine, coarse = layout.region_boxes(cfg, g)
        occ = []
        for c, box in enumerate((fine, coarse)):
            sh = layout.occupancy_shape(cfg, box)
            bits = (rng.random(sh[0] * sh[1] * sh[2]) < frac).astype(np.uint8)
            ctx.set_occupancy(g, c, bits)
            occ.append(bits)
        sel, t0, t1 = [], [], []
        for i in range(len(o)):
            for s in range(ns[i]):
                if reg[i, s] == g:
                    sel.append(i)
                    t0.append(te[i, s])
                    t1.append(tx[i, s])
        sel = np.array(sel)
        rid = sel.astype(np.uint64)
        cg, tg, dg_, casg = ctx.cascade_march(g, o[sel], d[sel], t0, t1, rid, jitter, 7)
        co, to, do, caso = om.cascade_march(g, occ[0], occ[1], o[sel], d[sel], t0, t1, rid, jitter, 7)
        assert np.array_equal(cg, co)
        assert np.array_equal(tg.view(np.uint64), to.view(np.uint64))
        assert np.array_equal(dg_.view(np.uint64), do.view(np.uint64))
        assert np.array_equal(casg, caso)
        assert (caso == 1).any() and (caso == 0).any()


# ------------------------------------------------------------------ stage 3
@pytest.mark.parametrize("table_log2,aspect", [(14, (1, 1, 1)), (19, (1.7, 1.0, 0.6)),
                                               (12, (4, 2, 1))])
def test_encode_indices_bit_exact(table_log2, aspect):
    cfg = small_cfg(1, 1, table_log2=table_log2, levels=16, nmax=2048, extent=aspect)
    ctx = dg.Context(cfg, device=0)
    om = OracleModel(cfg)
    p = layout.reference_like_init(cfg, 0, seed=3)
    rng = np.random.default_rng(4)
    p[:om_grid_floats(cfg)] = rng.uniform(-1, 1, om_grid_floats(cfg)).astype(np.float32)
    ctx.set_params(0, p)
    pts = rng.random((3000, 3))
    pts[:8] = [[0, 0, 0], [1, 1, 1], [0.5, 0.5, 0.5], [0.25, 0.5, 0.75], [1, 0, 1], [0, 1, 0],
               [1 / 15, 1 / 3, 2 / 7], [0.999999999, 1e-12, 0.5]]
    for cascade in (0, 1):
        fg, rg = ctx.encode(0, cascade, pts)
        fo, ro = om.encode(0, cascade, p, pts)
        assert np.array_equal(rg, ro)
        assert np.allclose(fg, fo, rtol=1e-5, atol=1e-6), np.abs(fg - fo).max()


def om_grid_floats(cfg):
    fine, _ = layout.region_boxes(cfg, 0)
    return sum(lv["rows"] * 2 for lv in layout.grid_levels(cfg, fine, cfg.fine_table_log2))


def test_encode_backward_matches_oracle():
    cfg = small_cfg(1, 1, table_log2=12, levels=8, nmax=128)
    ctx = dg.Context(cfg, device=0)
    om = OracleModel(cfg)
    p = layout.reference_like_init(cfg, 0)
    ctx.set_params(0, p)
    rng = np.random.default_rng(9)
    pts = rng.random((2000, 3))
    up = rng.uniform(-1, 1, (2000, 16)).astype(np.float32)
    ctx.zero_grads()
    ctx.encode_backward(0, 0, pts, up)
    g_gpu = ctx.get_grads(0)
    # oracle: adjoint via the field-free encode restatement, accumulated in fp64
    from oracle.bindings import oracle_lib  # noqa: F401
    ref = np.zeros_like(p)
    fine, _ = layout.region_boxes(cfg, 0)
    levels = layout.grid_levels(cfg, fine, cfg.fine_table_log2)
    _, rows = om.encode(0, 0, p, pts)
    off = 0
    offs = []
    for lv in levels:
        offs.append(off)
        off += lv["rows"] * 2
    # weights via encode of unit tables is complex; use the linearity identity instead:
    # <grad, t> == sum_i <up_i, encode(p_i; t)> for the tables t = p
    feats, _ = om.encode(0, 0, p, pts)
    lhs = float(np.dot(g_gpu[:off].astype(np.float64), p[:off]))
    rhs = float(np.sum(up.astype(np.float64) * feats))
    assert rel_err(lhs, rhs) < 1e-4
    assert np.count_nonzero(g_gpu[:off]) > 0


# ------------------------------------------------------------------ stage 4
@pytest.mark.parametrize("cascade", [0, 1])
def test_field_forward_backward(cascade, impl):
    cfg = small_cfg(1, 1, table_log2=14, levels=16, nmax=512)
    ctx = dg.Context(cfg, device=0)
    om = OracleModel(cfg)
    rng = np.random.default_rng(21 + cascade)
    p = layout.reference_like_init(cfg, 0, seed=5)
    # tables away from the ReLU kink (test_field.cpp:205-207)
    gf = om_grid_floats(cfg)
    p[:gf] = rng.uniform(-0.5, 0.5, gf).astype(np.float32)
    if cascade == 1:
        nf = layout.partition_arrays(cfg, 0)
        fine_size = sum(nf[:len(nf) // 2])
        _, coarse = layout.region_boxes(cfg, 0)
        cg = sum(lv["rows"] * 2 for lv in layout.grid_levels(cfg, coarse, cfg.coarse_table_log2))
        p[fine_size:fine_size + cg] = rng.uniform(-0.5, 0.5, cg).astype(np.float32)
    ctx.set_params(0, p)
    n = 3000
    pts = rng.random((n, 3))
    dirs = rng.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs = dirs.astype(np.float32).astype(np.float64)
    app = rng.uniform(-1, 1, (n, 16)).astype(np.float32).astype(np.float64)
    sg, cgpu = ctx.field_forward(0, cascade, pts, dirs, app)
    so, co = om.field_forward(0, cascade, p, pts, dirs, app)
    assert np.allclose(sg, so, rtol=1e-4, atol=1e-7), np.abs(sg / so - 1).max()
    assert np.allclose(cgpu, co, rtol=1e-4, atol=1e-7), np.abs(cgpu - co).max()
    dsig = rng.uniform(-1, 1, n).astype(np.float32)
    drgb = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    ctx.zero_grads()
    ctx.field_backward(0, cascade, pts, dirs, app, dsig, drgb)
    gg = ctx.get_grads(0).astype(np.float64)
    go = om.field_backward(0, cascade, p, pts, dirs, app, dsig, drgb)
    tol = 1e-4 if impl == "ffma" else 2e-3
    for arr in ctx.param_layout(0):
        if arr["cascade"] != cascade:
            continue
        a = slice(arr["offset"], arr["offset"] + arr["size"])
        if np.abs(go[a]).max() == 0:
            assert np.abs(gg[a]).max() == 0
            continue
        assert rel_l2(gg[a], go[a]) < tol, (arr, rel_l2(gg[a], go[a]))


# ------------------------------------------------------------------ composed step
@pytest.fixture(params=["tc", "ffma"])
def impl(request, monkeypatch):
    monkeypatch.setenv("DG_MLP", request.param)
    return request.param


def _pair(cfg, n_images=1, occupancy_fraction=None, seed=0, table_scale=None):
    app = app_rows(n_images)
    ctx = dg.Context(cfg, device=0)
    ctx.set_appearance(app)
    orc = OracleRun(cfg, app)
    inject(cfg, ctx, [orc], seed=seed, occupancy_fraction=occupancy_fraction,
           table_scale=table_scale)
    return ctx, orc, app


def _check_losses(sg, so):
    for k in LOSSES:
        assert rel_err(sg[k], so[k], 1e-9) < 1e-4, (k, sg[k], so[k])
    assert sg["rays"] == so["rays"] and sg["dropped_rays"] == so["dropped_rays"]
    assert abs(sg["lr"] - so["lr"]) < 1e-15


# Stated gradient tolerance (per parameter array, relative L2 against the fp64 oracle).
# tcgen05 (default): the oracle is tied to the GPU's ReLU decisions (see the module
# docstring); what remains is the split-bf16 backward GEMMs' 2^-17 operand error and fp32
# atomics: measured <= 2e-5 on every array in every state (tools/diag/diag_grad5.py).
# FFMA (untied): at the reference's init every ReLU pre-activation sits near 0, so a few
# (sample, unit) pairs flip between fp32 and fp64 (measured <= 1.4e-3 on grid levels at init,
# MLP <= 5e-5).  Which units flip depends on the features' last bits: with the forward's fp32
# corner weights (~1e-7 of a feature) the trained state measures ~1e-6 on three tilings and
# 7.7e-4 on one grid level of the 4x2 case (one flipped unit; identical with and without the
# spatial sample order, so it is the untied FFMA forward, not the schedule).
TOLS = {  # (impl, state) -> (grid tol, mlp tol)
    ("ffma", "init"): (3e-3, 2e-4), ("ffma", "trained"): (1.5e-3, 2e-4),
    ("tc", "init"): (1e-4, 1e-4), ("tc", "trained"): (1e-4, 1e-4),
}
MAX_TIES, TIE_Z = 64, 4e-6  # tied units per step and their largest |pre-activation|


def _step(ctx, orc, o, d, gt, img, step):
    sg, so, (ties, zmax) = tied_train_step(ctx, orc, o, d, gt, img, step)
    assert ties <= MAX_TIES and zmax <= TIE_Z, (ties, zmax)
    return sg, so


def _check_update(cfg, ctx, orc, p0, lr, tols=(1e-4, 1e-4), adam_frac=0.999):
    worst = {}
    for g in range(cfg.kx * cfg.ky):
        m_g, _, t_g = ctx.get_adam(g)
        m_o, _, t_o, ws = orc.adam(g)
        assert t_g == t_o
        grad_o = orc.grads(g)
        grad_g = m_g.astype(np.float64) / (1.0 - cfg.adam_beta1)  # first step: m = (1-b1) g
        for arr in ctx.param_layout(g):
            a = slice(arr["offset"], arr["offset"] + arr["size"])
            ref = grad_o[a]
            if np.abs(ref).max() == 0:
                assert np.abs(grad_g[a]).max() < 1e-20
                continue
            e = rel_l2(grad_g[a], ref)
            tol = tols[0] if arr["kind"] == 0 else tols[1]
            worst[arr["kind"]] = max(worst.get(arr["kind"], 0.0), e)
            assert e < tol, (g, arr, e, tol)
        dp_g = ctx.get_params(g).astype(np.float64) - p0[g]
        dp_o = orc.params(g) - p0[g]
        big = np.abs(grad_o) > 1e-6 * np.abs(grad_o).max()
        err = np.abs(dp_g - dp_o)[big]
        # sign flips of near-cancelling gradients are allowed on a tiny fraction
        assert np.mean(err <= 1e-3 * lr) > adam_frac, (g, np.mean(err <= 1e-3 * lr), err.max())
    print("grad rel-L2 by kind", worst)


@pytest.mark.parametrize("state", ["init", "trained"])
@pytest.mark.parametrize("kx,ky,gen,n", [(1, 1, "vertical", 2048), (2, 1, "independent", 2048),
                                         (2, 2, "independent", 2048), (4, 2, "drift", 2048)])
def test_train_step_parity(kx, ky, gen, n, state, impl):
    from .helpers import params_for
    cfg = small_cfg(kx, ky, table_log2=14, levels=16, nmax=512, divisor=64 * max(kx, ky))
    scale = None if state == "init" else 0.5
    ctx, orc, _ = _pair(cfg, table_scale=scale)
    o, d, gt, img = _rays(cfg, n, gen, seed=kx + 7 * ky)
    p0 = [params_for(cfg, g, table_scale=scale) for g in range(kx * ky)]
    sg, so = _step(ctx, orc, o, d, gt, img, 0)
    _check_losses(sg, so)
    # sample positions bit-exact against cascade_march of the same items
    om = OracleModel(cfg)
    ns, reg, te, tx = om.segment_rays(o, d)
    for g in range(kx * ky):
        rid, order, te_g, tx_g, cnt = ctx.last_item_data(g)
        want = [i for i in range(n) if g in reg[i, :ns[i]]]
        assert np.array_equal(rid, np.array(want, dtype=np.uint64))
        t_g, d_g, c_g = ctx.last_samples(g)
        occ = [np.ones(np.prod(layout.occupancy_shape(cfg, b)), np.uint8) for b in layout.region_boxes(cfg, g)]
        co, to, do, caso = om.cascade_march(g, occ[0], occ[1], o[rid.astype(int)], d[rid.astype(int)],
                                            te_g, tx_g, rid, 1, 0)
        assert np.array_equal(cnt, co)
        assert np.array_equal(t_g.view(np.uint64), to.view(np.uint64))
        assert np.array_equal(d_g.view(np.uint64), do.view(np.uint64))
    _check_update(cfg, ctx, orc, p0, sg["lr"], TOLS[(impl, state)])


def test_train_step_coarse_cascade_and_partial_occupancy(impl):
    cfg = small_cfg(2, 2, table_log2=13, levels=8, nmax=256, divisor=128,
                    inner=((0.3, 0.25, 0.0), (1.6, 1.8, 0.8)), occ_res=24)
    ctx, orc, _ = _pair(cfg, occupancy_fraction=0.6)
    o, d, gt, img = _rays(cfg, 3000, "random", seed=3)
    p0 = [layout.reference_like_init(cfg, g) for g in range(4)]
    sg, so = _step(ctx, orc, o, d, gt, img, 0)
    _check_losses(sg, so)
    assert any(ctx.last_items(g)[2] > 0 for g in range(4))  # coarse samples exist
    _check_update(cfg, ctx, orc, p0, sg["lr"], TOLS[(impl, "init")])


def test_train_step_wire_f32():
    cfg = small_cfg(2, 1, table_log2=13, levels=8, nmax=256, divisor=128, wire_f32=1)
    ctx, orc, _ = _pair(cfg)
    o, d, gt, img = _rays(cfg, 2000, "independent", seed=13)
    sg = ctx.train_step(o, d, gt, img, step=5)
    so = orc.train_step(o, d, gt, img, 5)
    _check_losses(sg, so)


def test_multi_step_tracks_oracle():
    cfg = small_cfg(2, 1, table_log2=13, levels=8, nmax=256, divisor=96)
    ctx, orc, _ = _pair(cfg)
    for step in range(3):
        o, d, gt, img = _rays(cfg, 1024, "independent", seed=100 + step)
        sg, so = _step(ctx, orc, o, d, gt, img, step)
        for k in LOSSES:  # state drifts slowly (Adam turns noise-level gradients into +-lr steps)
            assert rel_err(sg[k], so[k], 1e-9) < (1e-4 if step == 0 else 2e-3), (step, k)
    assert ctx.get_step() == 3


@pytest.mark.parametrize("t", [7, 300])
def test_adam_from_injected_moments(t, impl):
    """AdamState::step (train.cpp:91-115) past step 1: identical params, first / second moments
    and step counts injected on both sides, one training step at worker step t, then the new
    moments and parameters compared (the update is no longer -lr * sign(g))."""
    cfg = small_cfg(2, 1, table_log2=13, levels=8, nmax=256, divisor=96)
    ctx, orc, _ = _pair(cfg, table_scale=0.5)
    rng = np.random.default_rng(t)
    m0, v0, p0 = [], [], []
    for g in range(2):
        n = ctx.param_count(g)
        m = (rng.normal(size=n) * 1e-3).astype(np.float32)
        v = (rng.uniform(0.1, 4.0, n) * m.astype(np.float64) ** 2 + 1e-12).astype(np.float32)
        ctx.set_adam(g, m, v, t)
        orc.set_adam(g, m.astype(np.float64), v.astype(np.float64), t, t)
        m0.append(m.astype(np.float64))
        v0.append(v.astype(np.float64))
        p0.append(ctx.get_params(g).astype(np.float64))
    ctx.set_step(t)
    o, d, gt, img = _rays(cfg, 2048, "independent", seed=77)
    sg, so = _step(ctx, orc, o, d, gt, img, t)
    _check_losses(sg, so)
    lr = sg["lr"]
    for g in range(2):
        m_g, v_g, t_g = ctx.get_adam(g)
        m_o, v_o, t_o, _ = orc.adam(g)
        assert t_g == t_o == t + 1
        grad_o = orc.grads(g)
        for arr in ctx.param_layout(g):  # m = b1 m0 + (1 - b1) g, v = b2 v0 + (1 - b2) g^2
            a = slice(arr["offset"], arr["offset"] + arr["size"])
            assert rel_l2(m_g[a], m_o[a]) < 1e-4 and rel_l2(v_g[a], v_o[a]) < 1e-4, arr
        big = np.abs(grad_o) > 1e-6 * np.abs(grad_o).max()
        dp_g = ctx.get_params(g).astype(np.float64) - p0[g]
        dp_o = orc.params(g) - p0[g]
        err = np.abs(dp_g - dp_o)
        assert np.mean(err[big] <= 1e-3 * lr) >= 0.999, (g, np.mean(err[big] <= 1e-3 * lr))
        assert np.mean(err <= 1e-3 * lr) >= 0.999
        # the update is the bias-corrected ratio, not a sign step
        assert np.std(np.abs(dp_o[big]) / lr) > 0.05


def test_dropped_rays_and_empty_batch():
    cfg = small_cfg(2, 1, table_log2=12, levels=4, nmax=64)
    ctx, orc, _ = _pair(cfg)
    o, d, gt, img = _rays(cfg, 256, "independent", seed=1)
    o[::3] = [50.0, 50.0, 50.0]  # misses
    sg = ctx.train_step(o, d, gt, img, step=0)
    so = orc.train_step(o, d, gt, img, 0)
    _check_losses(sg, so)
    assert sg["dropped_rays"] == len(o[::3])
    st = ctx.train_step(o[:0], d[:0], gt[:0], img[:0], step=1)  # every worker still steps Adam
    assert st["rays"] == 0 and st["loss_rgb"] == 0.0
    _, _, t = ctx.get_adam(0)
    assert t == 2


def test_unknown_image_id_is_out_of_range():
    cfg = small_cfg(1, 1, table_log2=12, levels=4, nmax=64)
    ctx, _, _ = _pair(cfg)
    o, d, gt, img = _rays(cfg, 64, "vertical", seed=1)
    img[5] = 7
    with pytest.raises(dg.DGError) as e:
        ctx.train_step(o, d, gt, img, step=0)
    assert e.value.status == "DG_ERANGE"


# ------------------------------------------------------------------ render
@pytest.mark.parametrize("kx,ky,gen", [(1, 1, "vertical"), (2, 2, "independent"),
                                       (4, 2, "corner")])
def test_render_parity(kx, ky, gen):
    cfg = small_cfg(kx, ky, table_log2=14, levels=16, nmax=512, divisor=64 * max(kx, ky),
                    extent=(kx, ky, 0.5 if gen == "corner" else 1.0))
    ctx, orc, app = _pair(cfg, occupancy_fraction=0.8)
    o, d, _, _ = _rays(cfg, 3000, gen, seed=kx * ky)
    o[:10] = [[99.0, 99.0, 99.0]] * 10  # background rays
    rgb, T, depth = ctx.render(o, d, app[0])
    rgb_o, T_o, depth_o = orc.eval_rays(o, d, app[0])
    assert np.allclose(rgb, rgb_o, rtol=1e-4, atol=1e-6), np.abs(rgb - rgb_o).max()
    assert np.allclose(T, T_o, rtol=1e-4, atol=1e-6), np.abs(T - T_o).max()
    assert np.allclose(depth, depth_o, rtol=1e-4, atol=1e-5), np.abs(depth - depth_o).max()
    assert (T[:10] == 1.0).all() and (rgb[:10] == 0).all()


def test_init_reference_matches_reference_build():
    from oracle.bindings import RefRun, ref_available
    if not ref_available():
        pytest.skip("reference build not present")
    cfg = small_cfg(2, 1, table_log2=12, levels=6, nmax=128)
    ref = RefRun(cfg, app_rows(1))
    ctx = dg.Context(cfg, device=0)
    for g in range(2):
        ctx.init_reference(g)
        assert np.array_equal(ctx.get_params(g), ref.params(g).astype(np.float32))


# ------------------------------------------------------------------ occupancy update (§8f row 1)
@pytest.mark.parametrize("warmup", [4096, 4])
def test_occupancy_update_matches_reference_stream(warmup):
    """Steps 14, 15, 16 cross Worker::update_occupancy (worker.cpp:549-562).  The sampled
    cells and jitter points follow the reference's mt19937_64 stream, so bitfields agree except
    for cells whose density lies within fp32 resolution of the threshold."""
    cfg = small_cfg(2, 1, table_log2=12, levels=8, nmax=128, divisor=64, occ_res=16,
                    inner=((0.2, 0.1, 0.0), (1.7, 0.9, 0.9)))
    cfg.occ_warmup_steps = warmup
    cfg.occ_threshold_scale = 2.5  # threshold 1.5 vs sigma = exp(raw0): a mixed bitfield
    ctx, orc, _ = _pair(cfg, table_scale=0.5, occupancy_fraction=0.7)
    for step in (14, 15, 16):
        o, d, gt, img = _rays(cfg, 512, "random", seed=step)
        sg = ctx.train_step(o, d, gt, img, step=step)
        so = orc.train_step(o, d, gt, img, step)
        if step < 15:
            _check_losses(sg, so)
    mixed = False
    for g in range(2):
        for c, box in enumerate(layout.region_boxes(cfg, g)):
            sh = layout.occupancy_shape(cfg, box)
            n = sh[0] * sh[1] * sh[2]
            bg = ctx.get_occupancy(g, c)
            bo = orc.occupancy(g, c, n)
            assert np.mean(bg == bo) > 0.995, (g, c, np.mean(bg == bo))
            mixed |= 0 < bo.mean() < 1
    assert mixed


def test_train_step_nmax_8192(impl):
    """N_max = 8192 (the paper's setting, SURVEY §8 notation): finest levels far beyond the
    table, so every level above the dense ones hashes; losses and gradients within the bars."""
    cfg = small_cfg(1, 1, table_log2=14, levels=16, nmax=8192, divisor=96)
    ctx, orc, _ = _pair(cfg, table_scale=0.5)
    from .helpers import params_for
    o, d, gt, img = _rays(cfg, 1500, "independent", seed=21)
    p0 = [params_for(cfg, 0, table_scale=0.5)]
    sg, so = _step(ctx, orc, o, d, gt, img, 0)
    _check_losses(sg, so)
    shapes, modes, rows = ctx.grid_levels(0, 0)
    assert shapes.max() >= 8000 and modes[-1] == 1
    _check_update(cfg, ctx, orc, p0, sg["lr"], TOLS[(impl, "trained")])
