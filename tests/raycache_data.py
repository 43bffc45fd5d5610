"""Synthetic dataset for the ray-cache tests: cameras on a ring looking at the scene centre
(orthonormal camera-to-world rotations, det +1), images of different sizes, one val image."""
import numpy as np


def dataset(seed=5, sizes=((31, 17), (24, 40), (9, 9), (50, 33))):
    rng = np.random.default_rng(seed)
    poses, images = [], []
    for i, (w, h) in enumerate(sizes):
        ang = 2 * np.pi * i / len(sizes) + rng.uniform(-0.2, 0.2)
        pos = np.array([2.0 + 1.5 * np.cos(ang), 1.0 + 1.5 * np.sin(ang), 1.8 + rng.uniform(-0.1, 0.3)])
        fwd = np.array([2.0, 1.0, 0.3]) - pos
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, [0.0, 0.0, 1.0])
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd], axis=1)  # columns: camera x, y, z in world
        f = float(rng.uniform(0.8, 1.4)) * w
        poses.append(dict(image_id=100 + 7 * i, width=w, height=h, is_train=(i != 2), rotation=R,
                          translation=pos, fx=f, fy=f * rng.uniform(0.95, 1.05), cx=w / 2 + rng.uniform(-1, 1),
                          cy=h / 2 + rng.uniform(-1, 1)))
        images.append(rng.integers(0, 256, (h, w, 3), dtype=np.uint8))
    return poses, images
