"""Config 5: per-step cost of dynamic-sequence training on B200.

    python tools/bench_dynamic.py [--preset rotating-blob] [--rays 16] [--steps 20]

Frame 0 is trained with the static step for a few hundred steps, then frame 1 is timed
in both phases of `dynamic.train_frame`: transform-only (render + compositing backward
+ the input-gradient kernel; field frozen) and joint (+ field backward and Adam).  The
static fused step on the same state is timed alongside.  Prints one JSON line.
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
from paper_2212_05231_b200 import scene_io, trainer  # noqa: E402


def timed(fn, steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = [fn() for _ in range(steps)]
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="rotating-blob", choices=["rotating-blob", "translating-sphere"])
    ap.add_argument("--rays", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--views", type=int, default=24)
    ap.add_argument("--image", type=int, default=128)
    ap.add_argument("--frame0-steps", type=int, default=300)
    a = ap.parse_args()
    t0 = time.time()
    ds = scene_io.make_synthetic(a.preset, views=a.views, image_size=a.image, seed=0, frames=2)
    for t in range(2):
        ds.to_device(t)
    gen_s = time.time() - t0
    cfg = trainer.TrainConfig(batch_size=1 << a.rays, num_levels=16, table_size=2**19, seed=0, level_init=16,
                              total_steps=10 * a.frame0_steps)
    seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
    dyn.train_frame(seq, ds, 0, dyn.DynamicConfig(first_frame_steps=a.frame0_steps))
    st = seq.train
    ms_static, reps = timed(lambda: trainer.train_step(st, ds, time_index=0), a.steps)
    P_static = float(np.mean([r.sample_count for r in reps]))
    gt = dyn.GlobalTransform.identity()
    opt = dyn.TransformAdam()
    seq.frame = 0
    for _ in range(3):  # warm-up
        dyn.dynamic_step(seq, ds, 1, gt, opt, False, 1e-3)
    ms_tr, reps_tr = timed(lambda: dyn.dynamic_step(seq, ds, 1, gt, opt, False, 1e-3), a.steps)
    ms_joint, reps_j = timed(lambda: dyn.dynamic_step(seq, ds, 1, gt, opt, True, 1e-4), a.steps)
    m = cfg.batch_size
    print(json.dumps({
        "config": f"c5: {a.preset}, {a.views} views {a.image}px, 2^{a.rays} rays/step, 16-level 2^19 grid",
        "static_ms": ms_static, "static_rays_per_s": m / ms_static * 1e3, "static_P": P_static,
        "transform_only_ms": ms_tr, "transform_only_rays_per_s": m / ms_tr * 1e3,
        "transform_only_P": float(np.mean([r.sample_count for r in reps_tr])),
        "joint_ms": ms_joint, "joint_rays_per_s": m / ms_joint * 1e3,
        "joint_P": float(np.mean([r.sample_count for r in reps_j])),
        "recovered_T": gt.t.tolist(), "dataset_gen_s": gen_s,
    }))


if __name__ == "__main__":
    main()
