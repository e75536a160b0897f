"""Dynamic sequences on the device path (SPEC `dynamic`, config 5): a preset sequence
trained incrementally with `dynamic.train_frame`; reports per frame the recovered global
transform against the ground truth implied by the preset's motion (Eq. 11:
R_i = R'_{i-1} R'_i^T, T_i = R_i^T T'_{i-1} - T'_i for x_frame = R'_t x_c + T'_t),
held-out-view PSNR (a second camera set, seed 99) and the Eq. 12 chain identity.

    python tools/run_sequence.py [--preset translating-sphere] [--frames 10] [--views 12]
    SPEC acceptance #8: translating-sphere, 10 frames (the sphere leaves the box after ~15)
    config 5:           --preset rotating-blob --frames 100 --views 24
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
    ap.add_argument("--preset", default="translating-sphere", choices=["translating-sphere", "rotating-blob"])
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--views", type=int, default=12)
    ap.add_argument("--image", type=int, default=64)
    ap.add_argument("--frame0-steps", type=int, default=1500)
    ap.add_argument("--transform-steps", type=int, default=100)
    ap.add_argument("--frame-steps", type=int, default=1100)
    ap.add_argument("--lr-joint", type=float, default=1e-4, help="transform lr in the joint phase")
    ap.add_argument("--frame-lr-scale", type=float, default=0.3, help="field lr scale for frames > 0")
    ap.add_argument("--lr-transform", type=float, default=1e-3, help="transform lr, transform-only phase")
    ap.add_argument("--init-from-previous", action="store_true",
                    help="start gt_i at gt_{i-1} (constant-velocity prior) instead of identity")
    ap.add_argument("--transform-eikonal", action="store_true",
                    help="include the Eikonal term in the transform's gradient (off: colour loss only)")
    a = ap.parse_args()
    ds = scene_io.make_synthetic(a.preset, views=a.views, image_size=a.image, seed=0, frames=a.frames)
    ds_eval = scene_io.make_synthetic(a.preset, views=2, image_size=a.image, seed=99, frames=a.frames)
    for t in range(a.frames):
        ds.to_device(t)
    cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8,
                              max_resolution=128, init_radius=0.25, total_steps=2 * a.frame0_steps)
    dc = dyn.DynamicConfig(first_frame_steps=a.frame0_steps, transform_steps=a.transform_steps,
                           frame_steps=a.frame_steps, lr_transform_joint=a.lr_joint,
                           frame_lr_scale=a.frame_lr_scale, transform_eikonal=a.transform_eikonal,
                           lr_transform=a.lr_transform, init_from_previous=a.init_from_previous)
    seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
    rows = []
    for i in range(a.frames):
        torch.cuda.synchronize()
        t0 = time.time()
        dyn.train_frame(seq, ds, i, dc)
        torch.cuda.synchronize()
        secs = time.time() - t0
        gt = seq.transforms[-1]
        if i > 0:
            (Rp, Tp), (Rc, Tc) = ds.motion[i - 1], ds.motion[i]
            R_gt = Rp @ Rc.T
            want = R_gt.T @ Tp - Tc
        else:
            R_gt, want = np.eye(3), np.zeros(3)
        c = np.clip((np.trace(gt.rotation.T @ R_gt) - 1.0) / 2.0, -1.0, 1.0)
        rows.append({"frame": i, "T": gt.t.tolist(), "T_gt": want.tolist(),
                     "T_err": float(np.linalg.norm(gt.t - want)),
                     "angle_deg": float(np.rad2deg(np.linalg.norm(gt.w))),
                     "angle_gt_deg": float(np.rad2deg(np.arccos(np.clip((np.trace(R_gt) - 1) / 2, -1, 1)))),
                     "rot_err_deg": float(np.rad2deg(np.arccos(c))),
                     "psnr_heldout": heldout_psnr(seq, ds_eval, i, 8), "seconds": secs})
        print(json.dumps(rows[-1]), flush=True)
    # Eq. 12 identity over the sequence: chain == frame-by-frame Eq. 11
    x = np.random.default_rng(0).normal(size=(16, 3))
    y = x.copy()
    for gt in reversed(seq.transforms[1:]):
        y = gt.to_previous_frame(y)
    chain_err = float(np.abs(seq.chain.canonicalize(x) - y).max())
    print(json.dumps({"summary": {
        "preset": a.preset, "frames": a.frames,
        "max_T_err": max(r["T_err"] for r in rows[1:]) if a.frames > 1 else 0.0,
        "max_rot_err_deg": max(r["rot_err_deg"] for r in rows[1:]) if a.frames > 1 else 0.0,
        "psnr_frame0": rows[0]["psnr_heldout"], "min_psnr": min(r["psnr_heldout"] for r in rows),
        "chain_identity_max_err": chain_err, "steps_per_frame": a.frame_steps,
        "transform_steps": a.transform_steps, "lr_joint": a.lr_joint, "frame_lr_scale": a.frame_lr_scale,
        "views": a.views, "transform_eikonal": a.transform_eikonal, "lr_transform": a.lr_transform,
        "init_from_previous": a.init_from_previous,
        "mean_frame_seconds": float(np.mean([r["seconds"] for r in rows[1:]])) if a.frames > 1 else None}}))


if __name__ == "__main__":
    main()
