"""§8f row 2 on the GPU: dg_ray_cache_* against the oracle restatement (itself pinned bitwise
to the reference, tests/test_ray_cache.py): entries and drawn batches bit-exact (fp64 origin /
direction, colour as f32 of the reference's u8 / 255.0), and a training step fed the cache's
device batch equals one fed the same rays from host memory."""
import ctypes as C

import numpy as np
import pytest

from oracle.bindings import OracleRayCache
from paper_2405_04416_b200 import abi, dg

from .helpers import app_rows, inject, small_cfg
from .raycache_data import dataset

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("capacity,seed", [(500, 1), (37, 99)])
def test_ray_cache_matches_oracle(capacity, seed):
    poses, images = dataset()
    gpu = dg.RayCache(poses, images, capacity, seed, device=0)
    orc = OracleRayCache(poses, images, capacity, seed)
    for count in (300, 400, 3 * capacity + 5):
        gpu.refresh(count)
        orc.refresh(count)
        assert gpu.size() == orc.size()
        go, gd, ggt, gimg, gpix = gpu.snapshot()
        oo, od, ogt, oimg, opix = orc.snapshot()
        assert np.array_equal(_bits(go), _bits(oo))
        assert np.array_equal(_bits(gd), _bits(od))
        assert np.array_equal(ggt, ogt.astype(np.float32))
        assert np.array_equal(gimg, oimg) and np.array_equal(gpix, opix)
        # a drawn device batch
        b = gpu.draw(257)
        assert b.mem == abi.DG_MEM_DEVICE and b.n == 257
        bo = np.zeros((257, 3))
        bd = np.zeros((257, 3))
        bgt = np.zeros((257, 3), np.float32)
        bimg = np.zeros(257, np.uint32)
        rt = C.CDLL("libcudart.so.12")
        rt.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        for arr, ptr in ((bo, b.origin), (bd, b.dir), (bgt, b.color_gt), (bimg, b.image_id)):
            assert rt.cudaMemcpy(arr.ctypes.data, ptr, arr.nbytes, 2) == 0  # device -> host
        ro, rd, rgt, rimg, _ = orc.draw(257)
        assert np.array_equal(_bits(bo), _bits(ro)) and np.array_equal(_bits(bd), _bits(rd))
        assert np.array_equal(bgt, rgt.astype(np.float32)) and np.array_equal(bimg, rimg)


def test_train_step_from_cache_batch():
    poses, images = dataset()
    cfg = small_cfg(1, 1, table_log2=12, levels=8, nmax=128, divisor=64,
                    extent=(4.0, 2.0, 1.0))
    cache = dg.RayCache(poses, images, 4000, 3, device=0)
    orc = OracleRayCache(poses, images, 4000, 3)
    cache.refresh(4000)
    orc.refresh(4000)
    ids = sorted({p["image_id"] for p in poses})
    rows = app_rows(len(ids))
    a = dg.Context(cfg, device=0)
    b = dg.Context(cfg, device=0)
    for ctx in (a, b):
        ctx.set_appearance(rows.astype(np.float32), np.array(ids, np.uint32))
    inject(cfg, a, [b])
    batch = cache.draw(1024)
    st = abi.StepStats()
    assert b.train_step_raw(batch, 0, st) == 0
    o, d, gt, img, _ = orc.draw(1024)
    sa = a.train_step(o, d, gt.astype(np.float32), img, step=0)
    assert sa["rays"] == st.rays and sa["dropped_rays"] == st.dropped_rays
    for k in ("loss_rgb", "loss_transmittance", "loss_distortion"):
        assert abs(sa[k] - getattr(st, k)) <= 1e-6 * max(abs(sa[k]), 1e-12), k
    # same gradients (first Adam moment = (1 - b1) g) up to the atomics' summation order
    from .helpers import rel_l2
    assert rel_l2(b.get_adam(0)[0], a.get_adam(0)[0]) < 1e-5
