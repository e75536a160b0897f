"""Debug aid: transform gradient at frame 1 of translating-sphere vs finite differences."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05231_b200 import dynamic as dyn  # noqa: E402
from paper_2212_05231_b200 import renderer, scene_io, trainer  # noqa: E402

ds = scene_io.make_synthetic("translating-sphere", views=12, image_size=64, seed=0, frames=2)
cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8,
                          init_radius=0.25, total_steps=400)
seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
rep = dyn.train_frame(seq, ds, 0, dyn.DynamicConfig(first_frame_steps=300))
print("frame0 psnr", rep[-1].psnr, "loss", rep[-1].total)
st = seq.train
rng = np.random.default_rng(5)
batch = scene_io.sample_ray_batch(ds, 1, 8192, 0.9, rng)
batch0 = scene_io.sample_ray_batch(ds, 0, 8192, 0.9, np.random.default_rng(5))


def loss_at(gt, b, grad=False):
    ft = seq.chain.frame_transform(gt)
    if RESET:
        st.occ.ema.zero_()
    renderer.update_occupancy(st.occ, st.params, 8, point_transform=ft.point)
    rendered, rec = renderer.render_rays(b, st.params, st.occ, 8, point_transform=ft.point,
                                         dir_transform=ft.direction)
    color, eik, mse, dl_dc, dl_dsdf, dslog, dl_dn = dyn._cotangents(st, b, rendered, rec)
    out = (color, rec.sample_count, float(st.occ.bits.float().mean()))
    if grad:
        dx, dv = dyn.field_input_grads(st.params, rec.cache, dl_dc, dl_dsdf, None)
        v = torch.as_tensor(b.directions, device="cuda")[rec.ray_ids.long()]
        g = ft.param_gradient(rec.frame_positions, v, dx, dv)
        return out, g, rec.sample_count
    return out


RESET = False
for RESET in (False, True):
  print("RESET", RESET)
  for name, b in (("frame0", batch0), ("frame1", batch)):
    gt = dyn.GlobalTransform.identity()
    (l0, P, _), g, _ = loss_at(gt, b, True)
    fd = []
    for k in range(6):
        e = np.zeros(6)
        e[k] = 1e-3
        gp = dyn.GlobalTransform((gt.params + e)[:3], (gt.params + e)[3:])
        gm = dyn.GlobalTransform((gt.params - e)[:3], (gt.params - e)[3:])
        fd.append((loss_at(gp, b)[0] - loss_at(gm, b)[0]) / 2e-3)
    print(name, "P", P, "loss", l0)
    print("  analytic (color only)", np.array2string(g, precision=5))
    print("  finite diff          ", np.array2string(np.array(fd), precision=5))
    for tx in (-0.05, -0.025, 0.0, 0.025, 0.05):
        print("  loss at T_x", tx, loss_at(dyn.GlobalTransform(np.zeros(3), np.array([tx, 0, 0])), b))
