"""Diagnostic: per-level gradient error of one product train step vs the oracle,
next to the oracle's own 1e-7 self-sensitivity.  Usage (GPU box):
    NS2B_FIELD_FWD=simt NS2B_FIELD_BWD=tc python tools/diag_step.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "tests" / "golden"):
    sys.path.insert(0, str(p))
import numpy as np  # noqa: E402

from helpers import np_, product_state_from_oracle  # noqa: E402
from oracle import render as orender, scene as oscene, train as otrain  # noqa: E402
from paper_2212_05231_b200 import trainer as ptrain  # noqa: E402
from parity import max_err, rel_err  # noqa: E402
from test_gpu_parity import oracle_sensitivity  # noqa: E402

ds = oscene.make_synthetic("sphere", views=8, seed=0, image_size=64)
cfg = otrain.TrainConfig(batch_size=2048, num_levels=8, table_size=2**14, seed=0, level_init=8)
ost = otrain.TrainState.create(cfg)
orender.update_occupancy(ost.occ, ost.params, 8)
ost.step = 1
pst = product_state_from_oracle(ost)
b = oscene.sample_ray_batch(ds, 0, 2048, 0.9, np.random.default_rng(5))
sens = oracle_sensitivity(ost, ds, b)
tr = {}
ro = otrain.train_step(ost, ds, batch=b, trace=tr)
rp = ptrain.train_step(pst, ds, batch=b)
sdf_g, col_g, tab_g = pst.params.layout.views(pst.ws.grads)
og = tr["grads"]
tag = f"fwd={os.environ.get('NS2B_FIELD_FWD','tc')} bwd={os.environ.get('NS2B_FIELD_BWD','tc')}"
print(tag, "P", rp.sample_count, ro.sample_count, "loss", rp.total, ro.total)
gt = np_(tab_g)
for lv in range(8):
    print(f"  tables{lv}: err {rel_err(gt[lv], og.tables[lv]):.2e}/{max_err(gt[lv], og.tables[lv]):.2e}"
          f"  sens {sens[f'tables{lv}'][0]:.2e}/{sens[f'tables{lv}'][1]:.2e}")
for i in range(2):
    print(f"  sdf{i}: err {rel_err(np_(sdf_g[i]), og.sdf_layers[i]):.2e}  sens {sens[f'sdf{i}'][0]:.2e}")
for i in range(3):
    print(f"  color{i}: err {rel_err(np_(col_g[i]), og.color_layers[i]):.2e}  sens {sens[f'color{i}'][0]:.2e}")

# ---- intermediates of the same step
ws = pst.ws
P = rp.sample_count
rec = tr["records"]
def cmp(name, a, r):
    a = np.asarray(a, np.float64).reshape(r.shape); r = np.asarray(r, np.float64)
    d = np.abs(a - r)
    print(f"  {name}: relL2 {rel_err(a, r):.2e} maxabs {d.max():.2e} argmax {np.unravel_index(d.argmax(), d.shape)} n>1e-3rel {(d > 1e-3*np.abs(r).max()).sum()}")
cmp("sdf", np_(ws.sdf[:P]), rec.sdf)
cmp("colors", np_(ws.colors[:P]), rec.sample_colors)
cmp("dl_dsdf", np_(ws.dl_dsdf[:P]), tr["dl_dsdf"])
cmp("dl_dc", np_(ws.dl_dc[:P]), tr["dl_dc"])
ii = rec.interval_first
a_p = np_(ws.alphas[:P])[ii]
print("  alpha clamp-at-0 count (prod/oracle):", int((a_p == 0).sum()), int((rec.alphas == 0).sum()),
      " mismatched zero-status:", int(((a_p == 0) != (rec.alphas == 0)).sum()))
cmp("alphas", a_p, rec.alphas)
