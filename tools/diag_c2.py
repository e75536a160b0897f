"""Diagnose c2 table-gradient max errors: product field_backward fed the ORACLE's
per-sample cotangents for the c2 step, with cotangent variants, vs the oracle's
field_backward on the same inputs; per level relL2/max and the worst entries."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "tests" / "golden"):
    sys.path.insert(0, str(p))
from helpers import np_, product_params_from_oracle  # noqa: E402
from oracle import field as ofield, render as orender, scene as oscene, train as otrain  # noqa: E402
from paper_2212_05231_b200 import field as pfield, scene_io as pscene  # noqa: E402
from parity import max_err, rel_err  # noqa: E402

ds = pscene.make_synthetic_device("two-spheres", 49, 1600, 1200, 1.4 * 1200, torch.device("cuda"))
cfg = otrain.TrainConfig(batch_size=4096, num_levels=16, table_size=2**19, seed=0, level_init=16)
ost = otrain.TrainState.create(cfg, aabb=ds.scene_aabb)
orender.update_occupancy(ost.occ, ost.params, 16)
ost.step = 1
b = oscene.sample_ray_batch(ds, 0, 4096, 0.9, np.random.default_rng(21))
tr = {}
otrain.train_step(ost, ds, batch=b, trace=tr)  # (mutates ost; the trace holds the pre-step cache)
rec = tr["records"]
x, v = rec.positions if hasattr(rec, "positions") else None, None
cache = rec.cache
X = cache.x
V = cache.view_dirs
print("P", X.shape[0])
# fresh oracle params = the pre-step ones
cfg2 = otrain.TrainConfig(batch_size=4096, num_levels=16, table_size=2**19, seed=0, level_init=16)
o0 = otrain.TrainState.create(cfg2, aabb=ds.scene_aabb).params
pp = product_params_from_oracle(o0)
dl_dc, dl_dd, dl_dn = tr["dl_dc"], tr["dl_dsdf"], tr["dl_dn"]
oc = ofield.eval_field(o0, X, V, 16)
pc = pfield.eval_field(pp, X, V, 16)
for nm in ("d", "normals", "colors"):
    a, r = np_(getattr(pc, nm)), getattr(oc, nm)
    print(f"fwd {nm}: relL2 {rel_err(a, r):.2e} max {max_err(a, r):.2e}")
z = np.zeros_like
variants = {"full": (dl_dc, dl_dd, dl_dn), "no_dn": (dl_dc, dl_dd, None), "dd_only": (None, dl_dd, None),
            "dc_only": (dl_dc, None, None), "dn_only": (None, None, dl_dn)}
for name, (c, d, n) in variants.items():
    og = ofield.field_backward(o0, oc, dl_dc=c, dl_dd=d, dl_dn=n)
    pg = pfield.field_backward(pp, pc, dl_dc=c, dl_dd=d, dl_dn=n)
    gt = np_(pg.tables)
    worst = []
    for lv in range(16):
        r_, m_ = rel_err(gt[lv], og.tables[lv]), max_err(gt[lv], og.tables[lv])
        worst.append((m_, lv, r_))
    worst.sort(reverse=True)
    print(name, " ".join(f"L{lv}:{r_:.1e}/{m_:.1e}" for m_, lv, r_ in worst[:5]))
    m_, lv, _ = worst[0]
    dif = np.abs(gt[lv] - og.tables[lv]).ravel()
    idx = np.argsort(dif)[-5:]
    ref = og.tables[lv].ravel()
    print("   worst entries", [(int(i), float(ref[i]), float(gt[lv].ravel()[i])) for i in idx],
          "max|ref|", float(np.abs(ref).max()))

# ---- near-tie ReLU pre-activations (mask flips between fp32 BLAS and the tensor-core forward)
def margins(params, c):
    out = np.full(c.x.shape[0], np.inf)
    for net, t in ((params.sdf_net, c.sdf_trace), (params.color_net, c.color_trace)):
        a = t.x
        for h, act in zip(net.layers[:-1], t.activations):
            z = a.astype(np.float64) @ h.T.astype(np.float64)
            sc = np.abs(a).astype(np.float64) @ np.abs(h.T).astype(np.float64)
            out = np.minimum(out, (np.abs(z) / np.maximum(sc, 1e-30)).min(1))
            a = act
    return out


mg = margins(o0, oc)
for tau in (1e-7, 1e-6, 1e-5, 1e-4):
    sel = mg < tau
    c, d, n = dl_dc.copy(), dl_dd.copy(), dl_dn.copy()
    c[sel] = 0
    d[sel] = 0
    n[sel] = 0
    og = ofield.field_backward(o0, oc, dl_dc=c, dl_dd=d, dl_dn=n)
    pg = pfield.field_backward(pp, pc, dl_dc=c, dl_dd=d, dl_dn=n)
    gt = np_(pg.tables)
    w = max((max_err(gt[lv], og.tables[lv]), lv) for lv in range(16))
    r = max(rel_err(gt[lv], og.tables[lv]) for lv in range(16))
    print(f"tau {tau:.0e}: {sel.sum()} near-tie samples zeroed -> worst table max {w[0]:.2e} (L{w[1]}), worst relL2 {r:.2e}")
