"""NS2C checkpoints (reference `checkpoint.py:1-189`).

Byte-compatible with the reference format, so a run can resume here from a checkpoint
the reference wrote and vice versa:

    b"NS2C" | u32 version (1) | sections: 4-byte tag, u64 payload length, payload

Array sections are a u32-length-prefixed JSON header (`sort_keys`, compact separators)
followed by the raw little-endian arrays in header order.  Sections, in the reference's
order: GRID (tables + grid metadata), SDFN / COLN (MLP layers), SLOG (fp64 s_log),
ADAM (per-group m, v and step t, groups sorted by name), STEP (u64), RNGS (the numpy
bit-generator state as JSON), OCCG (occupancy ema fp64 + bits u8), CONF (TrainConfig
as JSON), then any caller-supplied extra sections.

The host layer (`CheckpointData`, `encode`, `decode`) is plain numpy; `save_checkpoint`
/ `load_checkpoint` move a device `trainer.TrainState` through it.
"""

from __future__ import annotations

import dataclasses
import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

MAGIC = b"NS2C"
VERSION = 1


def _json(obj) -> bytes:
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()


def _raw(a) -> bytes:
    a = np.ascontiguousarray(a)
    return a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()


def _spec(a):
    return {"shape": list(a.shape), "dtype": a.dtype.str.lstrip("<>=|")}


def _arrays_payload(meta, arrays) -> bytes:
    head = _json(meta)
    return b"".join([struct.pack("<I", len(head)), head] + [_raw(a) for a in arrays])


def _arrays_from(payload, key="arrays"):
    (n,) = struct.unpack_from("<I", payload, 0)
    meta = json.loads(payload[4:4 + n].decode())
    off = 4 + n
    out = []
    for spec in meta[key]:
        dt = np.dtype(spec["dtype"]).newbyteorder("<")
        count = int(np.prod(spec["shape"])) if spec["shape"] else 1
        a = np.frombuffer(payload, dtype=dt, count=count, offset=off)
        off += a.nbytes
        out.append(a.reshape(spec["shape"]).astype(dt.newbyteorder("=")))
    return meta, out


@dataclass
class CheckpointData:
    """Everything a checkpoint holds, as host (numpy / python) values."""

    tables: np.ndarray                     # (L, T, F) fp32
    grid_meta: dict                        # num_levels, table_size, features_per_level,
                                           # resolutions, aabb_min, aabb_extent
    sdf_layers: list                       # fp32 (n_l, n_{l-1})
    color_layers: list
    sharpness_log: np.ndarray              # fp64 (1,)
    adam: dict                             # name -> (m, v, t)
    step: int
    rng_state: dict                        # numpy bit_generator.state
    occ_resolution: int
    occ_aabb: list                         # [lo(3), hi(3)]
    occ_threshold: float
    occ_ema: np.ndarray                    # fp64 (G, G, G)
    occ_bits: np.ndarray                   # uint8 (G, G, G)
    config: dict                           # dataclasses.asdict(TrainConfig)
    extra: list = field(default_factory=list)  # [(tag, payload)]


def encode(d: CheckpointData) -> bytes:
    """Serialise (`checkpoint.py:76-114`)."""
    g = dict(d.grid_meta)
    g["arrays"] = [_spec(d.tables)]
    sections = [(b"GRID", _arrays_payload(g, [d.tables]))]
    for tag, layers in ((b"SDFN", d.sdf_layers), (b"COLN", d.color_layers)):
        sections.append((tag, _arrays_payload({"arrays": [_spec(h) for h in layers]}, layers)))
    sections.append((b"SLOG", _raw(np.asarray(d.sharpness_log, np.float64))))
    meta = {"keys": [], "steps": [], "arrays": []}
    arrays = []
    for key in sorted(d.adam):
        m, v, t = d.adam[key]
        meta["keys"].append(key)
        meta["steps"].append(int(t))
        meta["arrays"] += [_spec(m), _spec(v)]
        arrays += [m, v]
    sections.append((b"ADAM", _arrays_payload(meta, arrays)))
    sections.append((b"STEP", struct.pack("<Q", int(d.step))))
    sections.append((b"RNGS", _json(d.rng_state)))
    bits = np.asarray(d.occ_bits).astype(np.uint8)
    ometa = {"resolution": int(d.occ_resolution), "aabb": d.occ_aabb,
             "threshold": float(d.occ_threshold), "arrays": [_spec(d.occ_ema), _spec(bits)]}
    sections.append((b"OCCG", _arrays_payload(ometa, [d.occ_ema, bits])))
    sections.append((b"CONF", _json(d.config)))
    sections += list(d.extra)
    out = [MAGIC, struct.pack("<I", VERSION)]
    for tag, payload in sections:
        out += [tag, struct.pack("<Q", len(payload)), payload]
    return b"".join(out)


def split_sections(raw: bytes) -> dict:
    """tag -> payload (`checkpoint.py:117-131`, same errors)."""
    if raw[:4] != MAGIC:
        raise ValueError("not a checkpoint: bad magic")
    (version,) = struct.unpack_from("<I", raw, 4)
    if version != VERSION:
        raise ValueError(f"unsupported checkpoint version {version}")
    sections, off = {}, 8
    while off < len(raw):
        tag = raw[off:off + 4]
        (n,) = struct.unpack_from("<Q", raw, off + 4)
        off += 12
        sections[tag] = raw[off:off + n]
        off += n
    return sections


def read_sections(path) -> dict:
    return split_sections(Path(path).read_bytes())


_KNOWN = (b"GRID", b"SDFN", b"COLN", b"SLOG", b"ADAM", b"STEP", b"RNGS", b"OCCG", b"CONF")


def decode(raw: bytes) -> CheckpointData:
    """Parse (`checkpoint.py:134-189`) into host values."""
    sec = split_sections(raw)
    gmeta, (tables,) = _arrays_from(sec[b"GRID"])
    gmeta.pop("arrays")
    _, sdf = _arrays_from(sec[b"SDFN"])
    _, col = _arrays_from(sec[b"COLN"])
    slog = np.frombuffer(sec[b"SLOG"], dtype="<f8").astype(np.float64)
    ameta, arr = _arrays_from(sec[b"ADAM"])
    adam = {k: (arr[2 * i], arr[2 * i + 1], int(ameta["steps"][i])) for i, k in enumerate(ameta["keys"])}
    ometa, (ema, bits) = _arrays_from(sec[b"OCCG"])
    (step,) = struct.unpack("<Q", sec[b"STEP"])
    # extra sections keep their file order (dicts preserve insertion order)
    extra = [(t, p) for t, p in sec.items() if t not in _KNOWN]
    return CheckpointData(
        tables=tables, grid_meta=gmeta, sdf_layers=sdf, color_layers=col, sharpness_log=slog,
        adam=adam, step=int(step), rng_state=json.loads(sec[b"RNGS"].decode()),
        occ_resolution=int(ometa["resolution"]), occ_aabb=ometa["aabb"],
        occ_threshold=float(ometa["threshold"]), occ_ema=ema, occ_bits=bits,
        config=json.loads(sec[b"CONF"].decode()), extra=extra)


# ------------------------------------------------------------------ device state --
def _np(t):
    return t.detach().cpu().numpy().copy()


def from_state(state, extra_sections=None) -> CheckpointData:
    """Gather a device TrainState to host values (one D2H per array)."""
    p, occ = state.params, state.occ
    g = p.grid
    grid_meta = {"num_levels": g.num_levels, "table_size": g.table_size,
                 "features_per_level": g.features_per_level,
                 "resolutions": [int(r) for r in g.resolutions],
                 "aabb_min": g.aabb_min.tolist(), "aabb_extent": g.aabb_extent.tolist()}
    adam = {k: (_np(a.m), _np(a.v), a.t) for k, a in state.adam.items()}
    return CheckpointData(
        tables=_np(g.tables), grid_meta=grid_meta,
        sdf_layers=[_np(h) for h in p.sdf_net.layers], color_layers=[_np(h) for h in p.color_net.layers],
        sharpness_log=_np(p.sharpness_log).reshape(1), adam=adam, step=int(state.step),
        rng_state=state.rng.bit_generator.state, occ_resolution=occ.resolution,
        occ_aabb=[occ.lo.tolist(), occ.hi.tolist()], occ_threshold=occ.threshold,
        occ_ema=_np(occ.ema), occ_bits=_np(occ.bits).astype(np.uint8),
        config=dataclasses.asdict(state.config), extra=list(extra_sections or []))


def save_checkpoint(path, state, extra_sections=None):
    """Serialise a device `trainer.TrainState` (`checkpoint.py:76-114`)."""
    Path(path).write_bytes(encode(from_state(state, extra_sections)))


def to_state(d: CheckpointData, dp=None):
    """Rebuild a device TrainState from host values."""
    import torch

    from . import field as fieldmod
    from . import hash_encoding as enc
    from . import relu_mlp as mlp
    from . import renderer, trainer

    gm = d.grid_meta
    lo = np.asarray(gm["aabb_min"], np.float64)
    hi = lo + np.asarray(gm["aabb_extent"], np.float64)
    res = [int(r) for r in gm["resolutions"]]
    grid = enc.MultiResHashGrid(gm["num_levels"], res[0], res[-1], gm["features_per_level"],
                                gm["table_size"], (lo.tolist(), hi.tolist()),
                                tables=torch.from_numpy(np.ascontiguousarray(d.tables, np.float32)))
    grid.resolutions = np.asarray(res, np.int64)
    params = fieldmod.SdfFieldParams(grid, mlp.MlpWeights(d.sdf_layers), mlp.MlpWeights(d.color_layers),
                                     d.sharpness_log)
    cfg = trainer.TrainConfig(**d.config)
    occ = renderer.OccupancyGrid(d.occ_resolution, (tuple(d.occ_aabb[0]), tuple(d.occ_aabb[1])),
                                 d.occ_threshold)
    occ.ema.copy_(torch.from_numpy(np.ascontiguousarray(d.occ_ema, np.float64)))
    occ.bits.copy_(torch.from_numpy(np.ascontiguousarray(d.occ_bits).astype(np.uint8)))
    rng = np.random.default_rng(0)
    rng.bit_generator.state = d.rng_state
    state = trainer.TrainState(params, occ, cfg, rng, step=d.step, dp=dp)
    for key, (m, v, t) in d.adam.items():
        st = state.adam[key]
        st.m.copy_(torch.from_numpy(np.ascontiguousarray(m)).view_as(st.m))
        st.v.copy_(torch.from_numpy(np.ascontiguousarray(v)).view_as(st.v))
        st.t = int(t)
    return state


def load_checkpoint(path, dp=None):
    """(TrainState on the device, sections) from a checkpoint file (`checkpoint.py:134-189`)."""
    raw = Path(path).read_bytes()
    return to_state(decode(raw), dp=dp), split_sections(raw)
