"""Shared fixtures for the parity tests: identical injected state on both sides."""
import numpy as np

from paper_2405_04416_b200 import layout, workloads
from paper_2405_04416_b200.abi import default_config


def small_cfg(kx=1, ky=1, table_log2=14, levels=8, nmax=256, divisor=64, extent=None,
              inner=None, wire_f32=0, occ_res=32):
    ext = extent or (float(kx), float(ky), 1.0)
    cfg = workloads._box_config(ext, kx, ky, table_log2, divisor, levels=levels, nmax=nmax)
    cfg.occ_resolution = occ_res
    cfg.wire_f32 = wire_f32
    if inner is not None:
        for a in range(3):
            cfg.inner_lo[a] = inner[0][a]
            cfg.inner_hi[a] = inner[1][a]
    return cfg


def app_rows(n=1, dim=16, seed=3):
    return workloads.appearance_rows(dim, n, seed).astype(np.float32).astype(np.float64)


def params_for(cfg, g, seed=0, table_scale=None):
    """Reference-distribution parameters; table_scale re-draws the hash tables U[-s, s]
    (a trained-like state, as the reference's FD tests do, test_field.cpp:205-207)."""
    p = layout.reference_like_init(cfg, g, seed=seed)
    if table_scale is not None:
        rng = np.random.default_rng(777 + g + 31 * seed)
        for a in layout_arrays(cfg, g):
            if a["kind"] == 0:
                sl = slice(a["offset"], a["offset"] + a["size"])
                p[sl] = rng.uniform(-table_scale, table_scale, a["size"]).astype(np.float32)
    return p


def layout_arrays(cfg, g):
    sizes = layout.partition_arrays(cfg, g)
    L = cfg.grid_levels
    kinds = ([0] * L + [1, 2, 1, 2, 3, 4, 3, 4, 3, 4]) * 2
    out, off = [], 0
    for k, s in zip(kinds, sizes):
        out.append(dict(offset=off, size=s, kind=k))
        off += s
    return out


def inject(cfg, ctx, others, seed=0, occupancy_fraction=None, occ_seed=11, table_scale=None):
    """Same fp32-representable parameters (and occupancy bitfields) on every side."""
    rng = np.random.default_rng(occ_seed)
    P = cfg.kx * cfg.ky
    for g in range(P):
        p = params_for(cfg, g, seed=seed, table_scale=table_scale)
        if ctx is not None:
            ctx.set_params(g, p)
        for o in others:
            o.set_params(g, p)
        if occupancy_fraction is not None:
            fine, coarse = layout.region_boxes(cfg, g)
            for c, box in enumerate((fine, coarse)):
                sh = layout.occupancy_shape(cfg, box)
                bits = (rng.random(sh[0] * sh[1] * sh[2]) < occupancy_fraction).astype(np.uint8)
                if ctx is not None:
                    ctx.set_occupancy(g, c, bits)
                for o in others:
                    o.set_occupancy(g, c, bits)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def rel_err(a, b, floor=1e-12):
    return abs(a - b) / max(abs(b), floor)


def tied_train_step(ctx, orc, o, d, gt, img, step, partitions=None):
    """One training step on the GPU, then the oracle's on the same batch with the GPU's ReLU
    on/off decisions (tcgen05 path: the split-tf32 forward's masks) for every sample.  A unit
    whose fp64 pre-activation lies within fp32 noise of 0 may round to either side, and its
    whole gradient contribution switches with it; tying the decisions compares everything else
    at full precision.  Returns (gpu stats, oracle stats, (units decided against the fp64 sign,
    their largest |z|)) -- a test bounds the latter so only genuine near-ties are absorbed.
    On the FFMA path (no masks) the oracle runs untied."""
    from oracle.bindings import gpu_mask_words
    sg = ctx.train_step(o, d, gt, img, step=step)
    tied = []
    for g in (partitions if partitions is not None else ctx.local):
        try:
            words = gpu_mask_words(ctx.last_masks(g))
        except Exception:  # FFMA: no masks
            break
        orc.mask_override(g, words)
        tied.append(g)
    so = orc.train_step(o, d, gt, img, step)
    ovr = orc.override_stats()
    for g in tied:
        orc.mask_override(g, None)
    return sg, so, ovr
