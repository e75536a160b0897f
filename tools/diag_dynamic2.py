"""Debug aid: silhouette centroid of renders under a translation vs the frame masks."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05231_b200 import dynamic as dyn  # noqa: E402
from paper_2212_05231_b200 import renderer, scene_io, trainer  # noqa: E402

ds = scene_io.make_synthetic("translating-sphere", views=12, image_size=64, seed=0, frames=2)
cfg = trainer.TrainConfig(batch_size=4096, num_levels=8, table_size=2**14, seed=0, level_init=8, max_resolution=int(sys.argv[2]),
                          init_radius=0.25, total_steps=int(sys.argv[1]) * 2)
seq = dyn.SequenceState(trainer.TrainState.create(cfg, aabb=ds.scene_aabb))
rep = dyn.train_frame(seq, ds, 0, dyn.DynamicConfig(first_frame_steps=int(sys.argv[1])))
st = seq.train
print("sharpness", st.params.sharpness)
for t in (0, 1):
    fr = ds.frames_at(t)[0]
    ys, xs = np.nonzero(fr.mask > 0.5)
    print(f"frame {t} target mask centroid", xs.mean(), ys.mean(), xs.size)
    o, d = scene_io.generate_rays_grid(fr)
    for tx in (-0.05, 0.0, 0.05):
        ft = dyn.TransformChain().frame_transform(dyn.GlobalTransform(np.zeros(3), np.array([tx, 0.0, 0.0])))
        st.occ.ema.zero_()
        renderer.update_occupancy(st.occ, st.params, 8, point_transform=ft.point)
        b = scene_io.RayBatch(o, d, np.zeros_like(o), np.zeros(o.shape[0], bool))
        out, rec = renderer.render_rays(b, st.params, st.occ, 8, point_transform=ft.point,
                                        dir_transform=ft.direction)
        op = (1 - rec.transmittance).cpu().numpy().reshape(64, 64)
        ys, xs = np.nonzero(op > 0.5)
        img = out.cpu().numpy().reshape(64, 64, 3)
        err = float(((img - fr.image * fr.mask[..., None]) ** 2).mean())
        print(f"   T_x {tx:+.2f}: render centroid {xs.mean():.3f} {ys.mean():.3f} n {xs.size} mse {err:.5f}")


def grads(use_eik, n=20):
    out = []
    gt = dyn.GlobalTransform.identity()
    ft = seq.chain.frame_transform(gt)
    renderer.update_occupancy(st.occ, st.params, 8, point_transform=ft.point)
    rng = np.random.default_rng(11)
    for _ in range(n):
        b = scene_io.sample_ray_batch(ds, 1, 4096, 0.9, rng)
        rendered, rec = renderer.render_rays(b, st.params, st.occ, 8, point_transform=ft.point,
                                             dir_transform=ft.direction)
        color, eik, mse, dl_dc, dl_dsdf, dslog, dl_dn = dyn._cotangents(st, b, rendered, rec)
        dx, dv = dyn.field_input_grads(st.params, rec.cache, dl_dc, dl_dsdf, dl_dn if use_eik else None)
        v = torch.as_tensor(b.directions, device="cuda")[rec.ray_ids.long()]
        out.append(ft.param_gradient(rec.frame_positions, v, dx, dv))
    out = np.array(out)
    print("eik" if use_eik else "color-only", "mean", np.array2string(out.mean(0), precision=5),
          "std", np.array2string(out.std(0), precision=5))


grads(True)
grads(False)

import time
t0 = time.time()
rep1 = dyn.train_frame(seq, ds, 1, dyn.DynamicConfig(transform_steps=int(sys.argv[3]), frame_steps=int(sys.argv[4])))
print("frame1 T", seq.transforms[1].t, "angle deg", np.rad2deg(np.linalg.norm(seq.transforms[1].w)),
      "psnr", rep1[0].psnr, "->", rep1[-1].psnr, "time", time.time() - t0)
