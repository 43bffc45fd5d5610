"""Benchmark / parity workloads: BASELINE.json configs C1..C5 and the weak-scaling tiling.

Synthetic rays follow SURVEY.md §8(d): every ray joins a point `a` on the outer box's top
face to a point `b` on its bottom face, dir = normalize(b - a), origin = a - 0.25 * dir, so
each ray starts just above the top face.  Inner box == outer box, so every sample is
shaded by the fine cascade (the coarse cascade is still allocated and Adam-stepped).
Colour targets are U[0,1]^3, one appearance row (image 0) U[-1,1]^16, seed 1.
"""
from dataclasses import dataclass

import numpy as np

from .abi import default_config


@dataclass
class Workload:
    name: str
    cfg: object          # abi.RunConfig
    n_rays: int
    generator: str       # vertical | independent | drift | corner
    note: str = ""


def _box_config(outer_hi, kx, ky, table_log2, divisor, levels=16, nmax=2048):
    c = default_config()
    for a in range(3):
        c.inner_lo[a] = c.outer_lo[a] = 0.0
        c.inner_hi[a] = c.outer_hi[a] = float(outer_hi[a])
    c.kx, c.ky = kx, ky
    c.grid_levels = levels
    c.grid_features = 2
    c.base_resolution = 16
    c.max_resolution = nmax
    c.fine_table_log2 = table_log2
    c.coarse_table_log2 = 12
    c.appearance_dim = 16
    c.march_step_divisor = float(divisor)
    c.total_steps = 1000
    c.wire_f32 = 1  # benchmark mode: f32 partial payload (SURVEY 8d common settings)
    return c


def c1():
    """C1: 1 AABB, L=16 F=2 T=2^19, 64K vertical rays x exactly 128 samples (CPU-runnable)."""
    return Workload("C1", _box_config((1, 1, 1), 1, 1, 19, 128), 65536, "vertical")


def c2():
    """C2: 2 partitions along x, T=2^22, 256K rays, ~50% cross-boundary."""
    return Workload("C2", _box_config((2, 1, 1), 2, 1, 22, 193), 262144, "independent")


def c3():
    """C3: 2x2 tiling, T=2^24, 512K rays, ~75% cross."""
    return Workload("C3", _box_config((2, 2, 1), 2, 2, 24, 172), 524288, "independent")


def c4():
    """C4: 4x2 Rubble-like tiling, T=2^24, 1M rays, balanced reflected-drift generator."""
    return Workload("C4", _box_config((4, 2, 1), 4, 2, 24, 416), 1048576, "drift")


def c5():
    """C5: 4x2, T=2^24, worst case corner-to-corner rays (5 segments/ray), render-only."""
    return Workload("C5", _box_config((4, 2, 0.5), 4, 2, 24, 123), 1048576, "corner")


WEAK_TILINGS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}


def weak(n_gpus, rays_per_gpu=131072, table_log2=24):
    """Weak-scaling point of C4: G partitions on G GPUs, 128K rays per GPU,
    unit tiles, the same absolute march step 4/416 and the drift generator."""
    kx, ky = WEAK_TILINGS[n_gpus]
    cfg = _box_config((kx, ky, 1), kx, ky, table_log2, 104 * max(kx, ky))
    return Workload(f"C4-weak-{n_gpus}", cfg, rays_per_gpu * n_gpus, "drift",
                    note=f"{kx}x{ky} unit tiles, T=2^{table_log2}/partition, "
                         f"{rays_per_gpu} rays/GPU")


def by_name(name):
    return {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[name]()


def make_rays(cfg, n, generator, seed=1):
    """Returns origin (n,3) f64, dir (n,3) f64, color_gt (n,3) f32, image_id (n,) u32."""
    rng = np.random.default_rng(seed)
    lo = np.array(cfg.outer_lo[:], dtype=np.float64)
    hi = np.array(cfg.outer_hi[:], dtype=np.float64)
    ext = hi - lo
    top = np.empty((n, 3))
    bot = np.empty((n, 3))
    top[:, 2] = hi[2]
    bot[:, 2] = lo[2]
    if generator == "vertical":
        top[:, :2] = lo[:2] + rng.random((n, 2)) * ext[:2]
        bot[:, :2] = top[:, :2]
    elif generator == "independent":
        top[:, :2] = lo[:2] + rng.random((n, 2)) * ext[:2]
        bot[:, :2] = lo[:2] + rng.random((n, 2)) * ext[:2]
    elif generator == "drift":
        top[:, :2] = lo[:2] + rng.random((n, 2)) * ext[:2]
        b = top[:, :2] + rng.uniform(-1.0, 1.0, (n, 2))
        b = np.where(b < lo[:2], 2 * lo[:2] - b, b)
        b = np.where(b > hi[:2], 2 * hi[:2] - b, b)
        bot[:, :2] = b
    elif generator == "corner":
        top[:, 0] = lo[0] + rng.random(n) * 0.25
        top[:, 1] = lo[1] + rng.random(n) * 0.25
        bot[:, 0] = hi[0] - rng.random(n) * 0.25
        bot[:, 1] = hi[1] - rng.random(n) * 0.25
    elif generator == "random":
        # generic rays through the box from random outside points (parity stress)
        top = lo + rng.random((n, 3)) * ext
        bot = lo + rng.random((n, 3)) * ext
        top[:, 2] = hi[2] + 0.1
    else:
        raise ValueError(generator)
    v = bot - top
    length = np.sqrt(v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1] + v[:, 2] * v[:, 2])
    d = v / length[:, None]
    o = top - 0.25 * d
    gt = rng.random((n, 3)).astype(np.float32)
    img = np.zeros(n, dtype=np.uint32)
    return np.ascontiguousarray(o), np.ascontiguousarray(d), gt, img


def appearance_rows(dim=16, n_images=1, seed=1):
    rng = np.random.default_rng(seed + 1000)
    return rng.uniform(-1.0, 1.0, (n_images, dim))
