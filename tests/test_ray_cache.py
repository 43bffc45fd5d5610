"""§8f row 2 on CPU: the ray-cache restatement (oracle/dg_oracle.c or_ray_cache_*) against the
reference's own RayCache + make_pixel_ray (train.cpp:117-159, dataset.cpp:312-324), bitwise:
refreshes that fill, wrap and over-wrap the ring, and batches drawn with replacement."""
import numpy as np
import pytest

from oracle.bindings import OracleRayCache, RefRayCache, ref_available

from .raycache_data import dataset


def _same(a, b):
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) missing")
@pytest.mark.parametrize("capacity,seed", [(500, 1), (37, 99)])
def test_oracle_ray_cache_matches_reference(capacity, seed):
    poses, images = dataset()
    ref = RefRayCache(poses, images, capacity, seed)
    orc = OracleRayCache(poses, images, capacity, seed)
    for count in (300, 400, 3 * capacity + 5):
        ref.refresh(count)
        orc.refresh(count)
        assert ref.size() == orc.size() == min(capacity, ref.size())
        _same(ref.snapshot(), orc.snapshot())
        _same(ref.draw(257), orc.draw(257))
    o, d, c, img, pix = orc.snapshot()
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0)
    assert set(np.unique(img)) <= {p["image_id"] for p in poses if p["is_train"]}
    assert ((pix >> 32) == img).all()
