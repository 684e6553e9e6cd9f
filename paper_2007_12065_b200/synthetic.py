"""Seeded synthetic organized clouds for tests and benchmarks.

Scene definitions follow the reference's generators (flatpoly/synthetic.py:22-108:
a flat grid; a box room seen by a downward ceiling camera with two box
obstacles) and SURVEY.md Appendix B (the LiDAR range image of config C3).  The
arrays are not bit-identical to the reference's (different RNG draw order);
golden-vector parity uses inputs stored in tests/golden instead.
"""

from __future__ import annotations

import numpy as np


def flat_plane_opc(rows=20, cols=20, spacing=0.05, z=0.0, noise=0.0, seed=0):
    """Flat grid in the xy plane, +z mesh normals (synthetic.py:22-31 convention)."""
    g = np.random.default_rng(seed)
    r = np.arange(rows, dtype=np.float64)[:, None] * np.ones((1, cols))
    c = np.ones((rows, 1)) * np.arange(cols, dtype=np.float64)[None, :]
    out = np.empty((rows, cols, 3))
    out[..., 0] = c * spacing
    out[..., 1] = -r * spacing
    out[..., 2] = z
    if noise > 0:
        out[..., 2] += g.normal(0.0, noise, (rows, cols))
    return out


_DEFAULT_BOXES = (((-1.3, -1.3, 0.0), (-0.55, -0.55, 0.35)),
                  ((0.5, 0.3, 0.0), (1.25, 1.05, 0.5)))


def room_scene(n=250, noise=0.002, seed=0, half=2.0, wall_height=2.5, cam_height=2.4,
               fov_deg=120.0, boxes=_DEFAULT_BOXES):
    """(n, n, 3) range scan of a box room from a downward camera at the ceiling.

    Rays through an n x n pinhole grid (+y at the image top) hit the floor, four
    walls or two axis-aligned boxes; Gaussian range noise is added along each ray.
    """
    g = np.random.default_rng(seed)
    t_half = np.tan(np.deg2rad(fov_deg) / 2.0)
    sy = np.linspace(1.0, -1.0, n)[:, None] * np.ones((1, n))
    sx = np.ones((n, 1)) * np.linspace(-1.0, 1.0, n)[None, :]
    ray = np.stack([sx * t_half, sy * t_half, -np.ones((n, n))], axis=-1)
    ray /= np.sqrt((ray ** 2).sum(axis=-1, keepdims=True))
    eye = np.array([0.0, 0.0, cam_height])
    t_hit = np.full((n, n), np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        # floor z = 0, inside the room
        t = -eye[2] / ray[..., 2]
        x, y = eye[0] + t * ray[..., 0], eye[1] + t * ray[..., 1]
        ok = (t > 0) & (np.abs(x) <= half) & (np.abs(y) <= half)
        t_hit = np.where(ok & (t < t_hit), t, t_hit)
        # walls x = +-half, y = +-half up to wall_height
        for axis in (0, 1):
            for sgn in (1.0, -1.0):
                t = (sgn * half - eye[axis]) / ray[..., axis]
                other = eye[1 - axis] + t * ray[..., 1 - axis]
                z = eye[2] + t * ray[..., 2]
                ok = (t > 0) & (np.abs(other) <= half) & (z >= 0) & (z <= wall_height)
                t_hit = np.where(ok & (t < t_hit), t, t_hit)
        # boxes: slab test
        for lo, hi in boxes:
            lo, hi = np.asarray(lo), np.asarray(hi)
            t1 = (lo - eye) / ray
            t2 = (hi - eye) / ray
            tn = np.minimum(t1, t2).max(axis=-1)
            tf = np.maximum(t1, t2).min(axis=-1)
            ok = (tn <= tf) & (tn > 0)
            t_hit = np.where(ok & (tn < t_hit), tn, t_hit)
    rng_t = t_hit + g.normal(0.0, noise, (n, n))
    return eye + rng_t[..., None] * ray


def lidar_scan(rows=64, cols=1024, seed=3, noise=0.01, dropout=0.03, max_range=80.0):
    """Spinning-LiDAR range image with NaN gaps."""
    g = np.random.default_rng(seed)
    el = np.deg2rad(np.linspace(15.0, -25.0, rows))[:, None]
    az = np.linspace(-np.pi, np.pi, cols, endpoint=False)[None, :]
    ray = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az),
                    np.sin(el) * np.ones_like(az)], axis=-1)
    eye = np.array([0.0, 0.0, 1.73])
    t_hit = np.full((rows, cols), np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = -eye[2] / ray[..., 2]
        t_hit = np.where((t > 0) & (t < t_hit), t, t_hit)
        for axis, c in ((0, 15.0), (0, -15.0), (1, 8.0), (1, -8.0)):
            t = (c - eye[axis]) / ray[..., axis]
            z = eye[2] + t * ray[..., 2]
            ok = (t > 0) & (z >= 0) & (z <= 3.0) & (t < t_hit)
            t_hit = np.where(ok, t, t_hit)
    t_hit = t_hit + g.normal(0.0, noise, t_hit.shape)
    t_hit[(t_hit > max_range) | ~np.isfinite(t_hit)] = np.nan
    t_hit[g.random(t_hit.shape) < dropout] = np.nan
    return eye + t_hit[..., None] * ray


# ------------------------------------------------------------ benchmark configs
def config_c1():
    """C1: 250x250 room, lap 1 + bil 1 (BASELINE.json configs[0])."""
    return room_scene(n=250, noise=0.002, seed=11)


def config_c2(seed=2, dropout_seed=1000):
    """C2: 480x640 central crop of a 640 room with 2 % dropout (configs[1])."""
    o = room_scene(n=640, noise=0.002, seed=seed)[80:560, :].copy()
    o[np.random.default_rng(dropout_seed).random((480, 640)) < 0.02] = np.nan
    return o


def config_c3():
    """C3: 64x1024 LiDAR range image with NaN gaps (configs[2])."""
    return lidar_scan(64, 1024, seed=3)


def config_c4(seed=4):
    """C4: 1080x1920 central crop of a 1920 room (configs[3])."""
    return room_scene(n=1920, noise=0.002, seed=seed)[420:1500, :].copy()


def config_c5_base():
    """C5 base frame: the C2 crop before dropout (per-frame noise + dropout are added)."""
    return room_scene(n=640, noise=0.002, seed=2)[80:560, :].copy()


def config_c5_frames(count, base=None, start=0):
    """C5 frames: C2 base + per-frame N(0, 2 mm) noise + 2 % dropout (configs[4])."""
    if base is None:
        base = config_c5_base()
    out = np.empty((count,) + base.shape)
    for i in range(count):
        g = np.random.default_rng(1000 + start + i)
        f = base + g.normal(0.0, 0.002, base.shape)
        f[g.random(base.shape[:2]) < 0.02] = np.nan
        out[i] = f
    return out
