"""Config 4's single-GPU half: step time of the c2 workload along the
progressive level schedule (λ = 2 → 16, `trainer.py:123-126`), occupancy frozen after
the step-0 refresh so only λ changes.  Prints one JSON line per λ.

    python tools/bench_schedule.py [--steps-per-level 4]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2212_05231_b200 import renderer, trainer  # noqa: E402
from paper_2212_05231_b200.scene_io import DeviceRaySource, RayBatch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps-per-level", type=int, default=4)
    a = ap.parse_args()
    wl = bench.workload("c2")
    dev = torch.device("cuda", 0)
    ds = bench.make_dataset(wl, dev)
    m = wl["rays"]
    total = 15000
    cfg = trainer.TrainConfig(batch_size=m, num_levels=wl["levels"], table_size=wl["table"], seed=0,
                              level_init=2, total_steps=total, occupancy_update_every=1 << 30)
    st = trainer.TrainState.create(cfg)
    renderer.update_occupancy(st.occ, st.params, wl["levels"])
    src = DeviceRaySource(ds, m, 2, seed=1, device=dev)
    window = cfg.level_increment_fraction * total
    for lam in range(2, wl["levels"] + 1):
        st.step = int((lam - 2) * window) + 1  # first step with this λ (not a refresh step)
        b = RayBatch(*src.dev[lam % 2], None)
        trainer.train_step(st, ds, batch=b)  # warm-up at this λ
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = []
        for i in range(a.steps_per_level):
            st.step = int((lam - 2) * window) + 2 + i
            reps.append(trainer.train_step(st, ds, batch=RayBatch(*src.dev[i % 2], None)))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps_per_level
        assert all(r.level == lam for r in reps), [r.level for r in reps]
        print(json.dumps({"lambda": lam, "ms_per_step": ms, "rays_per_s": m / ms * 1e3,
                          "P": reps[-1].sample_count}), flush=True)


if __name__ == "__main__":
    main()
