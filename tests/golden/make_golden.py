"""Generates tests/golden/golden_small.npz by running the UNMODIFIED reference library
(oracle/_ref/libdistgrid_ref.so, built from /root/reference sources by oracle/Makefile) on a
small 2x2 configuration: one training step (losses, every parameter after Adam) from injected
state, one evaluation render, and the segment schedules.  Run from the repo root:
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import RefRun, ref_segment_rays  # noqa: E402
from paper_2405_04416_b200 import layout, workloads  # noqa: E402
from tests.helpers import app_rows, params_for, small_cfg  # noqa: E402


def main():
    cfg = small_cfg(2, 2, table_log2=10, levels=4, nmax=64, divisor=40,
                    inner=((0.3, 0.2, 0.0), (1.7, 1.8, 0.9)), occ_res=8)
    app = app_rows(1)
    ref = RefRun(cfg, app)
    o, d, gt, img = workloads.make_rays(cfg, 96, "random", seed=21)
    out = {"cfg": np.frombuffer(bytes(cfg), dtype=np.uint8), "app": app, "o": o, "d": d,
           "gt": gt, "img": img, "step": np.array(3)}
    rng = np.random.default_rng(2)
    for g in range(4):
        p = params_for(cfg, g, table_scale=0.3)
        ref.set_params(g, p)
        out[f"params0_{g}"] = p
        for c, (name, box) in enumerate(zip(("occ_fine", "occ_coarse"), layout.region_boxes(cfg, g))):
            sh = layout.occupancy_shape(cfg, box)
            bits = (rng.random(sh[0] * sh[1] * sh[2]) < 0.75).astype(np.uint8)
            ref.set_occupancy(g, c, bits)
            out[f"{name}_{g}"] = bits
    st = ref.train_step(o, d, gt, img, 3)
    out["losses"] = np.array([st["loss_rgb"], st["loss_transmittance"], st["loss_distortion"]])
    for g in range(4):
        out[f"params1_{g}"] = ref.params(g)
    out["eval_rgb"], out["eval_T"], out["eval_depth"] = ref.eval_rays(o, d, app[0])
    nseg, reg, te, tx = ref_segment_rays(cfg, o, d)
    out["nseg"], out["te"] = nseg, te
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "golden_small.npz"), **out)
    print("wrote golden_small.npz", st)


if __name__ == "__main__":
    main()
