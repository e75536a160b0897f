"""Diagnostic: forward-field error (tc vs oracle) on a train step's real samples."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "tests" / "golden"):
    sys.path.insert(0, str(p))
import numpy as np
from helpers import np_, product_params_from_oracle
from oracle import field as ofield, render as orender, scene as oscene, train as otrain
from paper_2212_05231_b200 import field as pfield

ds = oscene.make_synthetic("sphere", views=8, seed=0, image_size=64)
cfg = otrain.TrainConfig(batch_size=2048, num_levels=8, table_size=2**14, seed=0, level_init=8)
ost = otrain.TrainState.create(cfg)
orender.update_occupancy(ost.occ, ost.params, 8)
b = oscene.sample_ray_batch(ds, 0, 2048, 0.9, np.random.default_rng(5))
mr = orender.march_rays(b.origins, b.directions, ost.occ)
x = mr.positions
v = b.directions[mr.ray_ids]
oc = ofield.eval_field(ost.params, x, v, 8)
pp = product_params_from_oracle(ost.params)
pc = pfield.eval_field(pp, x, v, 8)
tag = f"fwd={os.environ.get('NS2B_FIELD_FWD','tc')}"
for name, a, r in (("d", np_(pc.d), oc.d), ("g", np_(pc.g), oc.g), ("n", np_(pc.normals), oc.normals),
                   ("c", np_(pc.colors), oc.colors)):
    a = a.astype(np.float64); r = r.astype(np.float64)
    rel = np.abs(a - r) / np.maximum(np.abs(r), 1e-30)
    print(f"{tag} {name}: relL2 {np.linalg.norm(a-r)/np.linalg.norm(r):.2e} maxabs {np.abs(a-r).max():.2e} "
          f"median elem rel {np.median(rel):.2e} p99 {np.percentile(rel, 99):.2e} mean signed {(a-r).mean():.2e}")
