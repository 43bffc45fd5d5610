"""The benchmark workloads (paper_2405_04416_b200/workloads.py) against the statistics SURVEY
§8(d) validated through the reference library, recomputed with the oracle on the CPU (small
samples): C1's vertical rays get exactly 128 samples each; the C4 weak-scaling point keeps
the absolute march step 4/416 at every GPU count; C5's corner rays cross kx + ky - 1 = 5
regions."""
import numpy as np

from oracle.bindings import OracleModel
from paper_2405_04416_b200 import layout, workloads


def _march_counts(cfg, o, d):
    om = OracleModel(cfg)
    ns, reg, te, tx = om.segment_rays(o, d)
    counts = np.zeros(len(o), np.int64)
    P = cfg.kx * cfg.ky
    for g in range(P):
        idx = [i for i in range(len(o)) if g in reg[i, :ns[i]]]
        if not idx:
            continue
        sl = [int(np.nonzero(reg[i, :ns[i]] == g)[0][0]) for i in idx]
        boxes = layout.region_boxes(cfg, g)
        occ = [np.ones(int(np.prod(layout.occupancy_shape(cfg, b))), np.uint8) for b in boxes]
        c, _, _, _ = om.cascade_march(g, occ[0], occ[1], o[idx], d[idx], te[idx, sl], tx[idx, sl],
                                      np.array(idx, np.uint64), 1, 0)
        counts[idx] += c
    return ns, counts


def test_c1_exactly_128_samples_per_ray():
    wl = workloads.c1()
    cfg = wl.cfg
    cfg.fine_table_log2 = 12  # the march does not depend on the table size
    o, d, _, _ = workloads.make_rays(cfg, 64, wl.generator, seed=1)
    ns, counts = _march_counts(cfg, o, d)
    assert (ns == 1).all()
    assert (counts == 128).all(), np.unique(counts)


def test_weak_points_keep_the_absolute_step():
    steps = set()
    for n in (1, 2, 4, 8):
        c = workloads.weak(n, table_log2=12).cfg
        ext = max(c.outer_hi[a] - c.outer_lo[a] for a in range(3))
        steps.add(round(ext / c.march_step_divisor, 12))
    assert steps == {round(4.0 / 416.0, 12)}


def test_c5_rays_cross_five_regions():
    wl = workloads.c5()
    cfg = wl.cfg
    cfg.fine_table_log2 = 12
    o, d, _, _ = workloads.make_rays(cfg, 32, wl.generator, seed=1)
    ns, _, _, _ = OracleModel(cfg).segment_rays(o, d)
    assert (ns == cfg.kx + cfg.ky - 1).all(), np.unique(ns)


def test_c4_drift_rays_samples_per_ray_near_128():
    wl = workloads.weak(1, table_log2=12)
    o, d, _, _ = workloads.make_rays(wl.cfg, 48, wl.generator, seed=2)
    _, counts = _march_counts(wl.cfg, o, d)
    assert 110 <= counts.mean() <= 140, counts.mean()
