"""Oracle: cameras, rays, ray-batch sampling and the analytic sphere scenes
(TEST INFRASTRUCTURE ONLY).  Restates `hashsdf/scene_io.py:29-378`; the synthetic
datasets are built in memory with the same uint8 quantisation the reference's PNG
round trip applies (so they equal `load_dataset(make_synthetic(...))`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LIGHT = np.array([0.35, 0.45, 0.82]) / np.linalg.norm([0.35, 0.45, 0.82])  # scene_io.py:222-223
AMBIENT = 0.3


@dataclass
class CameraFrame:
    """`scene_io.py:29-60`."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    pose: np.ndarray
    image: np.ndarray
    mask: np.ndarray
    time_index: int = 0


@dataclass
class MultiViewDataset:
    frames: list
    scene_aabb: tuple = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    num_time_steps: int = 1

    def frames_at(self, time_index):
        return [f for f in self.frames if f.time_index == time_index]


@dataclass
class RayBatch:
    origins: np.ndarray
    directions: np.ndarray
    target_colors: np.ndarray
    foreground_flags: np.ndarray

    @property
    def count(self):
        return self.origins.shape[0]


def generate_rays_grid(frame, pixels=None):
    """Pinhole rays through pixel centres (`scene_io.py:98-116`)."""
    if pixels is None:
        ys, xs = np.mgrid[0:frame.height, 0:frame.width]
        pixels = np.stack([xs.ravel(), ys.ravel()], axis=1)
    px = pixels[:, 0].astype(np.float64)
    py = pixels[:, 1].astype(np.float64)
    d_cam = np.stack([(px + 0.5 - frame.cx) / frame.fx, (py + 0.5 - frame.cy) / frame.fy,
                      np.ones_like(px)], axis=1)
    d = d_cam @ frame.pose[:3, :3].T
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.broadcast_to(frame.pose[:3, 3], d.shape).copy(), d


def sample_ray_batch(dataset, time_index, count, fg_fraction, rng):
    """floor(fg*count) foreground + rest background pixels, uniform over frames,
    targets image*mask (`scene_io.py:129-172`); identical rng consumption."""
    if count < 1:
        raise ValueError("count must be >= 1")
    frames = dataset.frames_at(time_index)
    if not frames:
        raise ValueError("empty foreground: no frames at this time index")
    fg, bg = [], []
    for k, f in enumerate(frames):
        ys, xs = np.nonzero(f.mask > 0.5)
        fg.append(np.stack([np.full_like(xs, k), xs, ys], axis=1))
        ys, xs = np.nonzero(f.mask <= 0.5)
        bg.append(np.stack([np.full_like(xs, k), xs, ys], axis=1))
    fg, bg = np.concatenate(fg), np.concatenate(bg)
    if fg.shape[0] == 0:
        raise ValueError("empty foreground")
    n_fg = int(np.floor(fg_fraction * count))
    n_bg = count - n_fg
    pick_fg = fg[rng.integers(0, fg.shape[0], size=n_fg)]
    if n_bg > 0 and bg.shape[0] == 0:
        pick_bg = fg[rng.integers(0, fg.shape[0], size=n_bg)]
        flags = np.ones(count, bool)
    else:
        pick_bg = bg[rng.integers(0, bg.shape[0], size=n_bg)]
        flags = np.concatenate([np.ones(n_fg, bool), np.zeros(n_bg, bool)])
    picks = np.concatenate([pick_fg, pick_bg])
    o, d, tgt = np.empty((count, 3)), np.empty((count, 3)), np.empty((count, 3))
    for k, f in enumerate(frames):
        sel = picks[:, 0] == k
        if not np.any(sel):
            continue
        o[sel], d[sel] = generate_rays_grid(f, picks[sel, 1:3])
        xs, ys = picks[sel, 1], picks[sel, 2]
        tgt[sel] = f.image[ys, xs] * f.mask[ys, xs, None]
    return RayBatch(o, d, tgt, flags)


def preset_scene(name, num_frames=1):
    """Static presets of `scene_io.py:229-263` (dynamic ones are out of scope)."""
    if name == "sphere":
        spheres = [(np.zeros(3), 0.5, np.array([0.85, 0.35, 0.25]))]
    elif name == "two-spheres":
        spheres = [(np.array([0.32, 0.0, 0.0]), 0.30, np.array([0.85, 0.35, 0.25])),
                   (np.array([-0.30, 0.05, 0.10]), 0.25, np.array([0.25, 0.45, 0.85]))]
    else:
        raise ValueError("unknown preset")
    return spheres, [(np.eye(3), np.zeros(3))] * num_frames


def trace_spheres(origins, dirs, spheres, rot, trans):
    """Exact first hit + Lambertian shading (`scene_io.py:269-300`)."""
    n = origins.shape[0]
    best = np.full(n, np.inf)
    which = np.full(n, -1)
    for si, (c, r, _) in enumerate(spheres):
        oc = origins - (rot @ c + trans)
        b = np.einsum("ij,ij->i", oc, dirs)
        disc = b * b - (np.einsum("ij,ij->i", oc, oc) - r * r)
        t = np.where(disc >= 0, -b - np.sqrt(np.maximum(disc, 0.0)), np.inf)
        t = np.where(t > 1e-6, t, np.inf)
        closer = t < best
        best = np.where(closer, t, best)
        which = np.where(closer, si, which)
    hit = np.isfinite(best)
    col = np.zeros((n, 3))
    for si, (c, r, albedo) in enumerate(spheres):
        sel = hit & (which == si)
        if not np.any(sel):
            continue
        p = origins[sel] + best[sel, None] * dirs[sel]
        nrm = ((p - (rot @ c + trans)) / r) @ rot
        lam = np.maximum(nrm @ LIGHT, 0.0)
        col[sel] = albedo[None, :] * (AMBIENT + (1 - AMBIENT) * lam)[:, None]
    return best, hit, np.clip(col, 0.0, 1.0)


def orbit_pose(azimuth, elevation, distance):
    """Camera-to-world looking at the origin (`scene_io.py:303-316`)."""
    eye = distance * np.array([np.cos(azimuth) * np.cos(elevation),
                               np.sin(azimuth) * np.cos(elevation), np.sin(elevation)])
    fwd = -eye / np.linalg.norm(eye)
    right = np.cross(fwd, np.array([0.0, 0.0, 1.0]))
    if np.linalg.norm(right) < 1e-6:
        right = np.array([1.0, 0.0, 0.0])
    right /= np.linalg.norm(right)
    pose = np.eye(4)
    pose[:3, 0], pose[:3, 1], pose[:3, 2], pose[:3, 3] = right, np.cross(fwd, right), fwd, eye
    return pose


def make_synthetic(preset, views=16, seed=0, image_size=128, width=None, height=None,
                   focal=None, distance=2.6):
    """In-memory `make_synthetic` (`scene_io.py:319-378`) for static presets; with
    width/height/focal given it builds the rectangular DTU-shaped variant."""
    spheres, motion = preset_scene(preset)
    w = int(width or image_size)
    h = int(height or image_size)
    f = float(focal) if focal is not None else image_size * 1.4
    cx, cy = w / 2.0, h / 2.0
    rng = np.random.default_rng(seed)
    elev = np.deg2rad(np.where(np.arange(views) % 2 == 0, 18.0, -12.0))
    azim = 2 * np.pi * np.arange(views) / views + rng.uniform(0, 2 * np.pi / views)
    rot, trans = motion[0]
    frames = []
    for v in range(views):
        pose = orbit_pose(azim[v], elev[v], distance)
        fr = CameraFrame(f, f, cx, cy, w, h, pose, None, None, 0)
        o, d = generate_rays_grid(fr)
        _, hit, col = trace_spheres(o, d, spheres, rot, trans)
        rgb8 = (col.reshape(h, w, 3) * 255).round().astype(np.uint8)
        fr.image = rgb8.astype(np.float64) / 255.0
        fr.mask = hit.reshape(h, w).astype(np.float64)
        frames.append(fr)
    return MultiViewDataset(frames)
