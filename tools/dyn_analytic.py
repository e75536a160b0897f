"""Transform pipeline check with an analytic field (no learning): render the rotating-blob's
frame-1 rays through render_rays(point_transform, dir_transform) with the exact canonical
SDF and shading (`params.evaluate` hook, renderer.py:234-244) over a scan of rotations
about z; the colour loss must be minimal at the true -6 deg."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05231_b200 import dynamic as dyn  # noqa: E402
from paper_2212_05231_b200 import renderer, scene_io  # noqa: E402


class Analytic:
    def __init__(self, spheres, sharpness=200.0):
        self.spheres, self.sharpness = spheres, sharpness
        light = np.asarray(scene_io.LIGHT, np.float64)
        self.light = torch.tensor(light, device="cuda")

    def evaluate(self, pos, view_dirs):
        p = torch.as_tensor(pos, device="cuda", dtype=torch.float64)
        best, col = None, None
        for c, r, albedo in self.spheres:
            cc = torch.tensor(c, device="cuda", dtype=torch.float64)
            v = p - cc
            dist = v.norm(dim=1)
            d = dist - r
            n = v / dist.clamp_min(1e-12)[:, None]
            lam = (n @ self.light).clamp_min(0.0)
            cl = torch.tensor(albedo, device="cuda", dtype=torch.float64) * (0.3 + 0.7 * lam)[:, None]
            if best is None:
                best, col = d, cl
            else:
                sel = d < best
                best = torch.where(sel, d, best)
                col = torch.where(sel[:, None], cl, col)
        return best.float(), col.clamp(0, 1).float()


ds = scene_io.make_synthetic("rotating-blob", views=12, image_size=64, seed=0, frames=2)
spheres, _ = scene_io.preset_scene("rotating-blob", 2)
params = Analytic(spheres)
occ = renderer.OccupancyGrid(128, ds.scene_aabb, 0.01)
occ.set_bits(np.ones((128, 128, 128), bool))
for frame in (1, 0):
    b = scene_io.sample_ray_batch(ds, frame, 1 << 15, 0.9, np.random.default_rng(5))
    out = []
    for a in np.linspace(-9, 3, 13):
        gt = dyn.GlobalTransform(np.array([0.0, 0.0, np.deg2rad(a)]), np.zeros(3))
        ft = dyn.TransformChain().frame_transform(gt)
        rendered, rec = renderer.render_rays(b, params, occ, 8, point_transform=ft.point, dir_transform=ft.direction)
        tgt = torch.as_tensor(b.target_colors, device="cuda", dtype=torch.float64)
        out.append((round(float(a), 1), round(float(((rendered - tgt) ** 2).mean()) * 1e4, 3)))
    print("frame", frame, out)
