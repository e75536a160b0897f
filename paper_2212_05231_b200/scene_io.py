"""Datasets, rays and ray-batch sampling (API of `hashsdf/scene_io.py`).

Host side (numpy), because the reference's training loop consumes its single seeded
generator here and only here (`trainer.py:287-289`); the fused step uploads the
sampled batch (pinned, asynchronous).  `make_synthetic` builds the analytic sphere
scenes in memory with the same uint8 quantisation the reference's PNG round trip
applies; `make_dtu_shaped` builds the rectangular 49-view 1600x1200 variant the
benchmark uses.  `DeviceRaySource` keeps a dataset's rays for a set of
pre-drawn pixel picks resident in HBM for the kernel-only benchmark leg.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

# pose orthonormality tolerance of CameraFrame.validate (`scene_io.py:26`)
POSE_ORTHO_TOL = 1e-4

LIGHT = np.array([0.35, 0.45, 0.82]) / np.linalg.norm([0.35, 0.45, 0.82])
AMBIENT = 0.3


@dataclass
class CameraFrame:
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

    def validate(self):
        """`scene_io.py:44-57`."""
        rot = self.pose[:3, :3]
        if (np.abs(rot @ rot.T - np.eye(3)).max() > POSE_ORTHO_TOL
                or abs(np.linalg.det(rot) - 1.0) > POSE_ORTHO_TOL):
            raise ValueError("invalid pose")
        if self.image.shape[:2] != (self.height, self.width) or self.mask.shape != (self.height, self.width):
            raise ValueError("inconsistent frame")
        if self.image.min() < 0 or self.image.max() > 1:
            raise ValueError("inconsistent frame: pixel values outside [0,1]")


@dataclass
class MultiViewDataset:
    frames: list
    scene_aabb: tuple = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    num_time_steps: int = 1

    def frames_at(self, time_index):
        return [f for f in self.frames if f.time_index == time_index]

    def __post_init__(self):
        self._pools = {}
        self._device_samplers = {}

    def to_device(self, time_index=0, device=None):
        """Keep this dataset's images, masks and pixel pools in HBM: sample_ray_batch
        (and so train_step) then builds its batches on the GPU (DeviceSampler)."""
        if time_index not in self._device_samplers:
            self._device_samplers[time_index] = DeviceSampler(self, time_index, device)
        return self._device_samplers[time_index]

    def pools(self, time_index):
        """(frames, fg pool, bg pool) cached per time index (scene_io.py:137-146)."""
        if time_index not in self._pools:
            frames = self.frames_at(time_index)
            fg, bg = [], []
            for k, f in enumerate(frames):
                ys, xs = np.nonzero(f.mask > 0.5)
                fg.append(np.stack([np.full_like(xs, k), xs, ys], axis=1))
                ys, xs = np.nonzero(f.mask <= 0.5)
                bg.append(np.stack([np.full_like(xs, k), xs, ys], axis=1))
            self._pools[time_index] = (frames, np.concatenate(fg) if fg else np.zeros((0, 3), np.int64),
                                       np.concatenate(bg) if bg else np.zeros((0, 3), np.int64))
        return self._pools[time_index]


@dataclass
class RayBatch:
    origins: object
    directions: object
    target_colors: object
    foreground_flags: object

    @property
    def count(self):
        return self.origins.shape[0]


def generate_ray(frame, px, py):
    """One world-space ray through pixel (px, py) (`scene_io.py:86-95`)."""
    if not (0 <= px < frame.width and 0 <= py < frame.height):
        raise ValueError("pixel out of range")
    d_cam = np.array([(px + 0.5 - frame.cx) / frame.fx, (py + 0.5 - frame.cy) / frame.fy, 1.0])
    d = frame.pose[:3, :3] @ d_cam
    d /= np.linalg.norm(d)
    return frame.pose[:3, 3].copy(), d


def project_point(frame, p_world):
    """World point -> (px, py), the inverse pinhole map (`scene_io.py:119-126`)."""
    rot = frame.pose[:3, :3]
    pc = rot.T @ (np.asarray(p_world) - frame.pose[:3, 3])
    return pc[0] / pc[2] * frame.fx + frame.cx - 0.5, pc[1] / pc[2] * frame.fy + frame.cy - 0.5


def scene_sdf(spheres, points):
    """Exact union-of-spheres SDF at (N,3) canonical points (`scene_io.py:261-266`)."""
    d = np.full(points.shape[0], np.inf)
    for center, radius, _ in spheres:
        d = np.minimum(d, np.linalg.norm(points - center, axis=1) - radius)
    return d


def load_dataset(path):
    """Dataset directory with `transforms.json` + PNGs (`scene_io.py:178-213`): RGBA
    alpha > 0.5 is the mask, RGB images get an all-ones mask; per-frame `time_index`."""
    import json
    from pathlib import Path

    from PIL import Image

    path = Path(path)
    manifest = path / "transforms.json"
    if not manifest.is_file():
        raise FileNotFoundError("dataset not found")
    meta = json.loads(manifest.read_text())
    frames, num_t = [], 1
    for entry in meta["frames"]:
        arr = np.asarray(Image.open(path / entry["file_path"])).astype(np.float64) / 255.0
        if arr.ndim == 2:
            arr = np.repeat(arr[:, :, None], 3, axis=2)
        if arr.shape[2] == 4:
            rgb, mask = arr[:, :, :3], (arr[:, :, 3] > 0.5).astype(np.float64)
        else:
            rgb, mask = arr[:, :, :3], np.ones(arr.shape[:2])
        t = int(entry.get("time_index", 0))
        num_t = max(num_t, t + 1)
        frame = CameraFrame(fx=float(meta["fl_x"]), fy=float(meta["fl_y"]), cx=float(meta["cx"]),
                            cy=float(meta["cy"]), width=int(meta["w"]), height=int(meta["h"]),
                            pose=np.asarray(entry["transform_matrix"], np.float64).reshape(4, 4),
                            image=rgb, mask=mask, time_index=t)
        frame.validate()
        frames.append(frame)
    aabb = tuple(map(tuple, meta.get("scene_aabb", [[-1, -1, -1], [1, 1, 1]])))
    return MultiViewDataset(frames, aabb, num_t)


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
    """floor(fg*count) foreground + background pixels uniformly over the frames,
    targets image*mask (`scene_io.py:129-172`); identical rng consumption."""
    if count < 1:
        raise ValueError("count must be >= 1")
    dev = getattr(dataset, "_device_samplers", {}).get(time_index)
    if dev is not None:
        return dev.sample(count, fg_fraction, rng)
    frames, fg, bg = dataset.pools(time_index)
    if not frames:
        raise ValueError("empty foreground: no frames at this time index")
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


def _rot_z(angle):
    c, s = np.cos(angle), np.sin(angle)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def preset_scene(name, num_frames=1):
    """Presets of `scene_io.py:230-257`: (spheres, per-frame motion), motion (R, T)
    mapping canonical -> frame coordinates, x_frame = R x_canonical + T."""
    static = [(np.eye(3), np.zeros(3))] * num_frames
    if name == "sphere":
        return [(np.zeros(3), 0.5, np.array([0.85, 0.35, 0.25]))], static
    if name == "two-spheres":
        return [(np.array([0.32, 0.0, 0.0]), 0.30, np.array([0.85, 0.35, 0.25])),
                (np.array([-0.30, 0.05, 0.10]), 0.25, np.array([0.25, 0.45, 0.85]))], static
    if name == "translating-sphere":
        return ([(np.zeros(3), 0.25, np.array([0.85, 0.35, 0.25]))],
                [(np.eye(3), np.array([0.05 * t, 0.0, 0.0])) for t in range(num_frames)])
    if name == "rotating-blob":
        return ([(np.array([0.25, 0.0, 0.0]), 0.28, np.array([0.85, 0.35, 0.25])),
                 (np.array([-0.18, 0.12, 0.14]), 0.20, np.array([0.25, 0.45, 0.85]))],
                [(_rot_z(np.deg2rad(6.0) * t), np.zeros(3)) for t in range(num_frames)])
    raise ValueError("unknown preset")


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
    """`scene_io.py:303-316`."""
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
                   focal=None, distance=2.6, chunk=1 << 20, frames=1):
    """In-memory `make_synthetic` (`scene_io.py:319-378`); with width/height/focal it
    builds a rectangular variant, with `frames` > 1 a dynamic sequence (the same
    cameras every frame, time_index t, the preset's per-frame rigid motion).  Images
    are uint8-quantised like the PNG round trip; the ground-truth motion is kept on
    the dataset as `.motion` (evaluation only, like ground_truth.json)."""
    spheres, motion = preset_scene(preset, frames)
    w = int(width or image_size)
    h = int(height or image_size)
    f = float(focal) if focal is not None else image_size * 1.4
    rng = np.random.default_rng(seed)
    elev = np.deg2rad(np.where(np.arange(views) % 2 == 0, 18.0, -12.0))
    azim = 2 * np.pi * np.arange(views) / views + rng.uniform(0, 2 * np.pi / views)
    out = []
    for t in range(frames):
        rot, trans = motion[t]
        out += _render_views(views, azim, elev, distance, f, w, h, spheres, rot, trans, t, chunk)
    ds = MultiViewDataset(out, num_time_steps=frames)
    ds.motion = motion
    return ds


def make_synthetic_device(preset, views, w, h, focal, device, seed=0, distance=2.6):
    """`make_synthetic` (`scene_io.py:319-378`, rectangular variant) with the per-pixel
    sphere tracing of every view on the GPU: the 49-view 1600x1200 DTU-shaped scene
    (94M pixels) in seconds instead of minutes.  Data preparation, not the training
    path; same cameras, uint8-quantised images and binary masks as `make_synthetic`."""
    spheres, motion = preset_scene(preset)
    rng = np.random.default_rng(seed)
    elev = np.deg2rad(np.where(np.arange(views) % 2 == 0, 18.0, -12.0))
    azim = 2 * np.pi * np.arange(views) / views + rng.uniform(0, 2 * np.pi / views)
    light = torch.tensor(LIGHT, dtype=torch.float64, device=device)
    ys, xs = torch.meshgrid(torch.arange(h, device=device, dtype=torch.float64),
                            torch.arange(w, device=device, dtype=torch.float64), indexing="ij")
    frames = []
    for v in range(views):
        pose = orbit_pose(azim[v], elev[v], distance)
        R = torch.tensor(pose[:3, :3], device=device)
        eye = torch.tensor(pose[:3, 3], device=device)
        dc = torch.stack([(xs.reshape(-1) + 0.5 - w / 2.0) / focal,
                          (ys.reshape(-1) + 0.5 - h / 2.0) / focal,
                          torch.ones(h * w, device=device, dtype=torch.float64)], 1)
        d = dc @ R.T
        d = d / torch.linalg.norm(d, dim=1, keepdim=True)
        best = torch.full((h * w,), float("inf"), device=device, dtype=torch.float64)
        which = torch.full((h * w,), -1, device=device, dtype=torch.int64)
        for si, (c, r, _) in enumerate(spheres):
            oc = eye - torch.tensor(c, device=device)
            b = d @ oc
            disc = b * b - (oc @ oc - r * r)
            t = torch.where(disc >= 0, -b - torch.sqrt(torch.clamp(disc, min=0.0)),
                            torch.full_like(b, float("inf")))
            t = torch.where(t > 1e-6, t, torch.full_like(t, float("inf")))
            closer = t < best
            best = torch.where(closer, t, best)
            which = torch.where(closer, torch.full_like(which, si), which)
        hit = torch.isfinite(best)
        col = torch.zeros((h * w, 3), device=device, dtype=torch.float64)
        for si, (c, r, albedo) in enumerate(spheres):
            sel = hit & (which == si)
            p = eye + best[sel, None] * d[sel]
            nrm = (p - torch.tensor(c, device=device)) / r
            lam = torch.clamp(nrm @ light, min=0.0)
            col[sel] = torch.tensor(albedo, device=device) * (0.3 + 0.7 * lam)[:, None]
        rgb8 = (col.clamp(0, 1) * 255).round().to(torch.uint8).reshape(h, w, 3).cpu().numpy()
        fr = CameraFrame(focal, focal, w / 2.0, h / 2.0, w, h, pose, rgb8.astype(np.float64) / 255.0,
                         hit.reshape(h, w).to(torch.float64).cpu().numpy(), 0)
        frames.append(fr)
    return MultiViewDataset(frames)


def _render_views(views, azim, elev, distance, f, w, h, spheres, rot, trans, t, chunk):
    frames = []
    for v in range(views):
        pose = orbit_pose(azim[v], elev[v], distance)
        fr = CameraFrame(f, f, w / 2.0, h / 2.0, w, h, pose, None, None, t)
        img = np.empty((h * w, 3), np.uint8)
        msk = np.empty(h * w, np.float64)
        ys, xs = np.mgrid[0:h, 0:w]
        pix = np.stack([xs.ravel(), ys.ravel()], axis=1)
        for s in range(0, h * w, chunk):
            o, d = generate_rays_grid(fr, pix[s:s + chunk])
            _, hit, col = trace_spheres(o, d, spheres, rot, trans)
            img[s:s + chunk] = (col * 255).round().astype(np.uint8)
            msk[s:s + chunk] = hit
        fr.image = img.reshape(h, w, 3).astype(np.float64) / 255.0
        fr.mask = msk.reshape(h, w)
        frames.append(fr)
    return frames


def make_dtu_shaped(views=49, width=1600, height=1200, seed=0, preset="two-spheres"):
    """Config-2 scene: 49 orbit cameras, 1600x1200, fx=fy=1.4*1200."""
    return make_synthetic(preset, views=views, seed=seed, width=width, height=height,
                          focal=1.4 * height)


class DeviceSampler:
    """`sample_ray_batch` with the dataset resident in HBM.

    The reference's rng draws stay on the host -- two `rng.integers` calls on the
    caller's generator, so the stream (and a checkpointed rng state) is identical --
    and only the pick indices (8 B per ray) are uploaded; pool lookup, pinhole rays and
    targets are one kernel (`ns2b_rays_from_picks`) over images (uint8), masks (0/1)
    and the foreground / background pixel pools kept on the device."""

    def __init__(self, dataset, time_index=0, device=None):
        from . import _lib

        self.time_index = time_index
        frames, fg, bg = dataset.pools(time_index)
        if not frames:
            raise ValueError("empty foreground: no frames at this time index")
        h, w = frames[0].height, frames[0].width
        if any(f.height != h or f.width != w for f in frames):
            raise NotImplementedError("device sampler needs frames of one size")
        imgs = np.stack([f.image for f in frames])
        u8 = np.rint(imgs * 255.0)
        if not (np.array_equal(u8 / 255.0, imgs) and u8.min() >= 0 and u8.max() <= 255):
            raise NotImplementedError("device sampler stores 8-bit images (image = u8 / 255)")
        masks = np.stack([f.mask for f in frames])
        if not np.all((masks == 0) | (masks == 1)):
            raise NotImplementedError("device sampler stores binary masks")
        dev = device or _lib.device()
        self.h, self.w, self.dev = h, w, dev
        self.images = torch.from_numpy(u8.astype(np.uint8)).to(dev)
        self.masks = torch.from_numpy(masks.astype(np.uint8)).to(dev)
        par = np.zeros((len(frames), 16))
        for k, f in enumerate(frames):
            par[k, :9] = f.pose[:3, :3].reshape(-1)
            par[k, 9:12] = f.pose[:3, 3]
            par[k, 12:] = (f.fx, f.fy, f.cx, f.cy)
        self.frames = torch.from_numpy(par).to(dev)
        hw = h * w
        if len(frames) * hw >= 1 << 31:  # flat pool indices are int32 on the device
            raise NotImplementedError(
                f"device sampler: {len(frames)} views of {w}x{h} exceed 2^31 pixels (int32 pool index)")

        def flat(pool):
            return torch.from_numpy((pool[:, 0] * hw + pool[:, 2] * w + pool[:, 1]).astype(np.int32)).to(dev)

        self.n_fg, self.n_bg = fg.shape[0], bg.shape[0]
        if self.n_fg == 0:
            raise ValueError("empty foreground")
        self.fg = flat(fg)
        self.bg = flat(bg) if self.n_bg else self.fg
        self._picks = None
        self._copied = None

    def _draw(self, count, fg_fraction, rng):
        """The reference's two rng draws (`scene_io.py:150-160`), host side."""
        if count < 1:
            raise ValueError("count must be >= 1")
        n_fg = int(np.floor(fg_fraction * count))
        n_bg = count - n_fg
        a = rng.integers(0, self.n_fg, size=n_fg)
        all_fg = n_bg > 0 and self.n_bg == 0
        b = rng.integers(0, self.n_fg if all_fg else self.n_bg, size=n_bg)
        return a, b, n_fg, all_fg

    def _build(self, a, b, o, d, t):
        """Upload picks [a (foreground pool) | b (background pool)] through a pinned
        staging buffer and build their rays into o, d, t (device, stream-ordered)."""
        from . import _lib

        count = a.shape[0] + b.shape[0]
        if self._copied is not None:
            self._copied.synchronize()  # the previous upload has left the pinned buffer
        if self._picks is None or self._picks.shape[0] < count:
            self._picks = torch.empty(max(count, 1), dtype=torch.int64).pin_memory()
        hp = self._picks[:count]
        hp[:a.shape[0]].copy_(torch.from_numpy(a))
        hp[a.shape[0]:].copy_(torch.from_numpy(b))
        picks = hp.to(self.dev, non_blocking=True)
        self._copied = torch.cuda.Event()
        self._copied.record()
        if count:
            _lib.call("ns2b_rays_from_picks", _lib.ptr(picks), count, a.shape[0], _lib.ptr(self.fg),
                      _lib.ptr(self.bg), _lib.ptr(self.frames), self.w, self.h, _lib.ptr(self.images),
                      _lib.ptr(self.masks), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), _lib.stream_ptr())
        self._last_picks = picks  # alive until the kernel has run (stream order)

    def sample(self, count, fg_fraction, rng):
        """RayBatch of device tensors; consumes `rng` exactly like sample_ray_batch."""
        a, b, n_fg, all_fg = self._draw(count, fg_fraction, rng)
        if all_fg:
            flags = torch.ones(count, dtype=torch.bool, device=self.dev)
        else:
            flags = torch.cat([torch.ones(n_fg, dtype=torch.bool, device=self.dev),
                               torch.zeros(count - n_fg, dtype=torch.bool, device=self.dev)])
        o = torch.empty((count, 3), dtype=torch.float64, device=self.dev)
        d, t = torch.empty_like(o), torch.empty_like(o)
        self._build(a, b, o, d, t)
        return RayBatch(o, d, t, flags)

    def draw_key(self, count, fg_fraction):
        """What `_draw` depends on besides the rng: a draw made ahead is valid for any
        later call with the same key."""
        return (self.n_fg, self.n_bg, int(count), float(fg_fraction))

    def sample_into(self, count, fg_fraction, rng, o, d, t, rank=0, world=1, draw=None):
        """Rays rank, rank + world, ... of the `count`-ray global batch (the interleaved
        data-parallel shard, `parallel.shard_slice`) into caller buffers of
        `parallel.shard_size(count, rank, world)` rows.  The rng is consumed for the whole
        global batch, as every rank (and the reference) does; only the shard's picks
        (8 B per ray) are uploaded and only its rays are built.  `draw` is a `_draw`
        result made ahead from the same rng (then `rng` is not consumed here)."""
        a, b, n_fg, all_fg = draw if draw is not None else self._draw(count, fg_fraction, rng)
        if all_fg:  # background picks index the foreground pool: one pool
            a, b = np.concatenate([a, b])[rank::world], b[:0]
        else:
            a, b = a[rank::world], b[(rank - n_fg) % world::world]
        n = a.shape[0] + b.shape[0]
        if o.shape[0] != n:
            raise ValueError(f"sample_into: buffers hold {o.shape[0]} rays, the shard has {n}")
        self._build(np.ascontiguousarray(a), np.ascontiguousarray(b), o, d, t)


class DeviceRaySource:
    """Pre-drawn ray batches resident in HBM (benchmark inputs): `n_batches` batches of
    `count` rays sampled with the reference sampler semantics from one seeded rng."""

    def __init__(self, dataset, count, n_batches, fg_fraction=0.9, seed=0, device=None,
                 pin_host=True):
        rng = np.random.default_rng(seed)
        self.host = []
        self.dev = []
        # on a device the batches come from the device sampler (origins and targets
        # bit-identical to the host sampler, directions within 2 ulp of the host BLAS
        # order; ~200x faster at 2^18 rays); the host copies feed the e2e leg
        sampler = DeviceSampler(dataset, 0, device) if device is not None else None
        for _ in range(n_batches):
            if sampler is not None:
                b = sampler.sample(count, fg_fraction, rng)
                db = (b.origins, b.directions, b.target_colors)
                hb = tuple(t.cpu() for t in db)
                self.dev.append(db)
            else:
                b = sample_ray_batch(dataset, 0, count, fg_fraction, rng)
                hb = tuple(torch.from_numpy(np.ascontiguousarray(a, np.float64)) for a in
                           (b.origins, b.directions, b.target_colors))
            if pin_host:
                hb = tuple(t.pin_memory() for t in hb)
            self.host.append(hb)

    def __len__(self):
        return len(self.host)
