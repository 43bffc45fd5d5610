"""Host-side layout math shared by the Python binding and the tests.

Mirrors the C++ runtime's setup code (csrc/host.cpp) and the reference formulas:
  GridConfig::level_resolution  grid.cpp:56-63
  grid_shape                    grid.cpp:65-73
  HashGrid ctor (mode, rows)    grid.cpp:90-105
  FieldParams widths            field.cpp:189-201
  split_regions                 partition.cpp:206-252
"""
import math

import numpy as np


def level_resolution(levels, base, maxr, level):
    if levels == 1:
        return base
    growth = math.exp((math.log(float(maxr)) - math.log(float(base))) / float(levels - 1))
    v = float(base) * math.pow(growth, float(level))
    # std::llround: round half away from zero
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def grid_shape(aspect, n):
    s = max(aspect[0], max(aspect[1], aspect[2]))
    return tuple(int(math.ceil(a / s * float(n))) for a in aspect)


def planes(lo, hi, k):
    return [lo if i == 0 else hi if i == k else lo + (hi - lo) * float(i) / float(k)
            for i in range(k + 1)]


def region_boxes(cfg, g):
    kx, ky = cfg.kx, cfg.ky
    xp = planes(cfg.inner_lo[0], cfg.inner_hi[0], kx)
    yp = planes(cfg.inner_lo[1], cfg.inner_hi[1], ky)
    ix, iy = g % kx, g // kx
    fine = ((xp[ix], yp[iy], cfg.inner_lo[2]), (xp[ix + 1], yp[iy + 1], cfg.inner_hi[2]))
    coarse = ((cfg.outer_lo[0] if ix == 0 else xp[ix], cfg.outer_lo[1] if iy == 0 else yp[iy],
               cfg.outer_lo[2]),
              (cfg.outer_hi[0] if ix == kx - 1 else xp[ix + 1],
               cfg.outer_hi[1] if iy == ky - 1 else yp[iy + 1], cfg.outer_hi[2]))
    return fine, coarse


def grid_levels(cfg, box, table_log2):
    lo, hi = box
    aspect = [hi[a] - lo[a] for a in range(3)]
    T = 1 << table_log2
    out = []
    for l in range(cfg.grid_levels):
        n = level_resolution(cfg.grid_levels, cfg.base_resolution, cfg.max_resolution, l)
        shp = grid_shape(aspect, n)
        vox = shp[0] * shp[1] * shp[2]
        hashed = vox > T
        out.append(dict(shape=shp, hashed=hashed, rows=T if hashed else vox))
    return out


def field_arrays(cfg, box, table_log2):
    """Sizes of FieldParams::parameter_arrays in order (field.cpp:203-208)."""
    F = cfg.grid_features
    sizes = [lv["rows"] * F for lv in grid_levels(cfg, box, table_log2)]
    enc = cfg.grid_levels * F
    cin = 15 + 16 + cfg.appearance_dim
    sizes += [64 * enc, 64, 16 * 64, 16]
    sizes += [64 * cin, 64, 64 * 64, 64, 3 * 64, 3]
    return sizes


def partition_arrays(cfg, g):
    fine, coarse = region_boxes(cfg, g)
    return field_arrays(cfg, fine, cfg.fine_table_log2) + \
        field_arrays(cfg, coarse, cfg.coarse_table_log2)


def partition_param_count(cfg, g):
    return int(sum(partition_arrays(cfg, g)))


def occupancy_shape(cfg, box):
    lo, hi = box
    return grid_shape([hi[a] - lo[a] for a in range(3)], cfg.occ_resolution)


def reference_like_init(cfg, g, seed=0):
    """Random parameters with the reference's distributions (tables U[-1e-4,1e-4],
    Xavier-uniform weights, zero biases; grid.cpp:103, mlp.cpp:47-51), numpy stream.
    Values are rounded to fp32 so both oracle (fp64) and device (fp32) see identical state."""
    rng = np.random.default_rng(1_000_003 * (seed + 1) + g)
    fine, coarse = region_boxes(cfg, g)
    out = []
    for box, tl in ((fine, cfg.fine_table_log2), (coarse, cfg.coarse_table_log2)):
        F = cfg.grid_features
        for lv in grid_levels(cfg, box, tl):
            out.append(rng.uniform(-1e-4, 1e-4, lv["rows"] * F))
        enc = cfg.grid_levels * F
        cin = 15 + 16 + cfg.appearance_dim
        for (i, o) in ((enc, 64), (64, 16)):
            b = math.sqrt(6.0 / (i + o))
            out += [rng.uniform(-b, b, i * o), np.zeros(o)]
        for (i, o) in ((cin, 64), (64, 64), (64, 3)):
            b = math.sqrt(6.0 / (i + o))
            out += [rng.uniform(-b, b, i * o), np.zeros(o)]
    return np.concatenate(out).astype(np.float32).astype(np.float64)
