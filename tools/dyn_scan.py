"""Where does the translating-sphere transform estimate settle, and why?  (SPEC #8 diagnostic)

Trains frame 0 like tools/run_sequence.py, then for frame 1 (ground truth T = (-0.05, 0, 0))
  (a) scans the frozen field's colour / Eikonal loss over T_x on one fixed large batch;
  (b) runs the transform-only phase from identity with the Eikonal term in the transform
      gradient (as dynamic_step does) and without it, printing the trajectory.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05231_b200 import dynamic as dyn  # noqa: E402
from paper_2212_05231_b200 import renderer, scene_io, trainer  # noqa: E402


def main():
    f0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
    preset = sys.argv[2] if len(sys.argv) > 2 else "translating-sphere"
    views = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    image = int(sys.argv[4]) if len(sys.argv) > 4 else 64
    frames = 2
    ds = scene_io.make_synthetic(preset, views=views, image_size=image, seed=0, frames=frames)
    for t in range(frames):
        ds.to_device(t)
    cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8,
                              max_resolution=128, init_radius=0.25 if preset == "translating-sphere" else 0.4,
                              total_steps=2 * f0)
    seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
    dc = dyn.DynamicConfig(first_frame_steps=f0)
    dyn.train_frame(seq, ds, 0, dc)
    st = seq.train
    level = trainer.level_schedule(st.step, cfg)
    out = {"preset": preset, "frame0_steps": f0, "views": views, "image": image,
           "sharpness": st.params.sharpness, "scan": [], "scan_frame0": []}
    rot = preset != "translating-sphere"
    grid = np.deg2rad(np.linspace(-9, 3, 13)) if rot else np.linspace(-0.08, -0.02, 13)
    for frame, key in ((1, "scan"), (0, "scan_frame0")):
        batch = scene_io.sample_ray_batch(ds, frame, 1 << 16, cfg.fg_fraction, np.random.default_rng(5))
        for tx in (grid if frame == 1 else grid - grid[len(grid) * 3 // 4]):  # frame 0: around identity
            gt = (dyn.GlobalTransform(np.array([0.0, 0.0, tx]), np.zeros(3)) if rot
                  else dyn.GlobalTransform(np.zeros(3), np.array([tx, 0.0, 0.0])))
            ft = seq.chain.frame_transform(gt)
            occ = renderer.OccupancyGrid(cfg.occupancy_resolution, ds.scene_aabb, cfg.occupancy_threshold)
            renderer.update_occupancy(occ, st.params, level, point_transform=ft.point)
            rendered, rec = renderer.render_rays(batch, st.params, occ, level, point_transform=ft.point,
                                                 dir_transform=ft.direction)
            color, eik, mse, *_ = dyn._cotangents(st, batch, rendered, rec)
            # the same with the view directions left in frame space (isolates the colour
            # network's view dependence from the geometry)
            rendered2, rec2 = renderer.render_rays(batch, st.params, occ, level, point_transform=ft.point)
            color_v0 = dyn._cotangents(st, batch, rendered2, rec2)[0]
            out[key].append({"tx": round(float(tx), 4), "color": color, "eikonal": eik,
                             "total": color + cfg.eikonal_weight * eik, "color_frame_view_dirs": color_v0})
    print(json.dumps(out))
    # (b) transform-only trajectories, with and without the Eikonal term in its gradient
    for use_eik in (True, False):
        gt = dyn.GlobalTransform.identity()
        opt = dyn.TransformAdam()
        traj = []
        st_step = st.step
        for k in range(400):
            dyn.dynamic_step(seq, ds, 1, gt, opt, False, 1e-3, transform_eikonal=use_eik)
            if k % 50 == 49:
                traj.append([round(float(v), 5) for v in (gt.w if rot else gt.t)])
        st.step = st_step
        print(json.dumps({"eikonal_in_transform_grad": use_eik, "T_trajectory_every_50": traj}))


if __name__ == "__main__":
    main()
