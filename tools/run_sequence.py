"""SPEC acceptance #8 on the device path: a translating-sphere sequence (Δ = 0.05 / frame)
trained incrementally with `dynamic.train_sequence`; reports per-frame recovered
translations vs ground truth, held-out-view PSNR (a second camera set, seed 99) and the
Eq. 12 chain identity.

    python tools/run_sequence.py [--frames 10] [--frame0-steps 1500] [--frame-steps 1100]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2212_05231_b200 import dynamic as dyn  # noqa: E402
from paper_2212_05231_b200 import renderer, scene_io, trainer  # noqa: E402


def heldout_psnr(seq, ds_eval, frame, level):
    """Full-frame PSNR of the frame's held-out views, rendered through the chain."""
    chain = seq.chain
    errs = []
    for fr in ds_eval.frames_at(frame):
        o, d = scene_io.generate_rays_grid(fr)
        b = scene_io.RayBatch(o, d, np.zeros_like(o), np.zeros(o.shape[0], bool))
        ft = dyn.FrameTransform(dyn.TransformChain(chain.R, chain.T), dyn.GlobalTransform.identity())
        occ = renderer.OccupancyGrid(seq.train.config.occupancy_resolution, ds_eval.scene_aabb,
                                     seq.train.config.occupancy_threshold)
        renderer.update_occupancy(occ, seq.train.params, level, point_transform=ft.point)
        out, _ = renderer.render_rays(b, seq.train.params, occ, level, point_transform=ft.point,
                                      dir_transform=ft.direction)
        tgt = (fr.image * fr.mask[..., None]).reshape(-1, 3)
        errs.append(float(((out.cpu().numpy() - tgt) ** 2).mean()))
    return trainer.psnr_from_mse(float(np.mean(errs)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--views", type=int, default=12)
    ap.add_argument("--image", type=int, default=64)
    ap.add_argument("--frame0-steps", type=int, default=1500)
    ap.add_argument("--transform-steps", type=int, default=100)
    ap.add_argument("--frame-steps", type=int, default=1100)
    ap.add_argument("--lr-joint", type=float, default=1e-4, help="transform lr in the joint phase")
    ap.add_argument("--frame-lr-scale", type=float, default=0.3, help="field lr scale for frames > 0")
    a = ap.parse_args()
    ds = scene_io.make_synthetic("translating-sphere", views=a.views, image_size=a.image, seed=0, frames=a.frames)
    ds_eval = scene_io.make_synthetic("translating-sphere", views=2, image_size=a.image, seed=99, frames=a.frames)
    for t in range(a.frames):
        ds.to_device(t)
    cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8,
                              max_resolution=128, init_radius=0.25, total_steps=2 * a.frame0_steps)
    dc = dyn.DynamicConfig(first_frame_steps=a.frame0_steps, transform_steps=a.transform_steps,
                           frame_steps=a.frame_steps, lr_transform_joint=a.lr_joint,
                           frame_lr_scale=a.frame_lr_scale)
    seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
    rows = []
    for i in range(a.frames):
        torch.cuda.synchronize()
        t0 = time.time()
        dyn.train_frame(seq, ds, i, dc)
        torch.cuda.synchronize()
        secs = time.time() - t0
        gt = seq.transforms[-1]
        want = -(ds.motion[i][1] - ds.motion[i - 1][1]) if i > 0 else np.zeros(3)
        rows.append({"frame": i, "T": gt.t.tolist(), "T_gt": want.tolist(),
                     "T_err": float(np.linalg.norm(gt.t - want)),
                     "angle_deg": float(np.rad2deg(np.linalg.norm(gt.w))),
                     "psnr_heldout": heldout_psnr(seq, ds_eval, i, 8), "seconds": secs})
        print(json.dumps(rows[-1]), flush=True)
    # Eq. 12 identity over the sequence: chain == frame-by-frame Eq. 11
    x = np.random.default_rng(0).normal(size=(16, 3))
    y = x.copy()
    for gt in reversed(seq.transforms[1:]):
        y = gt.to_previous_frame(y)
    chain_err = float(np.abs(seq.chain.canonicalize(x) - y).max())
    print(json.dumps({"summary": {
        "frames": a.frames, "max_T_err": max(r["T_err"] for r in rows[1:]) if a.frames > 1 else 0.0,
        "psnr_frame0": rows[0]["psnr_heldout"], "min_psnr": min(r["psnr_heldout"] for r in rows),
        "chain_identity_max_err": chain_err, "steps_per_frame": a.frame_steps,
        "transform_steps": a.transform_steps, "lr_joint": a.lr_joint, "frame_lr_scale": a.frame_lr_scale,
        "mean_frame_seconds": float(np.mean([r["seconds"] for r in rows[1:]])) if a.frames > 1 else None}}))


if __name__ == "__main__":
    main()
