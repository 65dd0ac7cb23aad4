"""Scene containers, the WRFC checkpoint format, and seeded synthetic scenes.

The on-disk format is the reference's single-file checkpoint "WRFC"
(/root/reference/proj/src/checkpoint.cpp:51-141): header, a 3-entry section
table, the WRF2 Gaussian section (splat.cpp:711-736), the WRFD deform section
(deform.cpp:328-384) and a JSON trailer (checkpoint.cpp:36-49). Files written
here load unchanged in the reference (`train::load_checkpoint`) and in the
native library (`swr_scene_create_wrfc`).

Synthetic scenes follow SURVEY.md section 8(d): centres U[-2,2]^2, l1/l3 in
[0.5, 4] cells, l2 in [-0.5, 0.5] l1, logits U[-3,3], responses N(0, 0.05),
trunk weights U[+-1/sqrt(cols)] (deform.cpp:96-101) and head weights calibrated
so the residuals are non-trivial (RMS centre offset ~ 1 cell, RMS attenuation
offset ~ 0.05, RMS response offset ~ RMS response). numpy's PCG64 is the RNG;
both sides of every parity test load the same bytes, so the draw order of the
reference Rng does not matter here.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

PI = math.pi
TRUNK = 8
SKIP = (2, 4, 6)  # 0-based trunk layers that see [h, x] (deform.cpp:41)


@dataclass
class Scene:
    H: int
    W: int
    center_raw: np.ndarray  # [n, 2] f32 (elevation, azimuth), pre-tanh
    cholesky: np.ndarray    # [n, 3] f32 (l1, l2, l3)
    atten_logit: np.ndarray  # [n] f32
    response: np.ndarray    # [n, 2] f32
    width: int = 156
    bands_c: int = 10
    bands_p: int = 6
    weights: list = field(default_factory=list)  # 11 x [rows, cols] f32, WRFD order
    biases: list = field(default_factory=list)   # 11 x [rows] f32
    cutoff: float = 3.0
    tile: int = 16
    bbox_min: tuple = (0.0, 0.0, 0.0)
    bbox_max: tuple = (1.0, 1.0, 1.0)
    rssi_cal: tuple | None = None  # (slope, intercept) of an RSSI model (tasks.cpp:131-150)

    @property
    def n(self) -> int:
        return int(self.atten_logit.shape[0])

    @property
    def input_dim(self) -> int:
        return 2 * (2 * self.bands_c + 1) + 3 * (2 * self.bands_p + 1)

    def layer_shapes(self):
        D, Wd = self.input_dim, self.width
        shapes = [(Wd, D if i == 0 else (Wd + D if i in SKIP else Wd)) for i in range(TRUNK)]
        return shapes + [(2, Wd), (2, Wd), (1, Wd)]

    def cell_el(self) -> float:
        return (PI / 2.0) / self.H

    def cell_az(self) -> float:
        return (2.0 * PI) / self.W


# ------------------------------------------------------------------ WRFC I/O

def _config_json(sc: Scene) -> dict:
    # keys of train_config_to_json (config.cpp:84-101)
    return {
        "primitives": sc.n, "bands_center": sc.bands_c, "bands_position": sc.bands_p,
        "width": sc.width, "cutoff_radius": float(sc.cutoff), "tile": sc.tile,
        "lr_gaussian": 1e-2, "lr_mlp": 8e-3, "lambda1": 0.7, "coarse_iters": 10000,
        "fine_iters": 100000, "anneal_scale": 1.0, "anneal_threshold": 10000, "seed": 1234,
    }


def write_wrfc(path: str, sc: Scene) -> None:
    f32 = lambda a: np.ascontiguousarray(a, dtype="<f4").tobytes()
    wrf2 = b"WRF2" + struct.pack("<III", 1, sc.n, 0) + f32(sc.center_raw) + f32(sc.cholesky) \
        + f32(sc.atten_logit) + f32(sc.response)
    wrfd = b"WRFD" + struct.pack("<IIIII", 1, 11, sc.width, sc.bands_c, sc.bands_p)
    for w in sc.weights:
        wrfd += struct.pack("<II", w.shape[0], w.shape[1])
    for w, b in zip(sc.weights, sc.biases):
        wrfd += f32(w) + f32(b)
    tj = {
        "config": _config_json(sc), "iteration": 0, "manifest_hash": "0000000000000000",
        "grid": {"n_elevation": sc.H, "n_azimuth": sc.W},
        "bbox_min": list(map(float, sc.bbox_min)), "bbox_max": list(map(float, sc.bbox_max)),
    }
    if sc.rssi_cal is not None:  # save_rssi_model's extra keys (tasks.cpp:131-137)
        tj["rssi_slope"], tj["rssi_intercept"] = float(sc.rssi_cal[0]), float(sc.rssi_cal[1])
    trailer = json.dumps(tj, separators=(",", ":")).encode()
    head = 16 + 3 * 16
    offs = [head, head + len(wrf2), head + len(wrf2) + len(wrfd)]
    sizes = [len(wrf2), len(wrfd), len(trailer)]
    with open(path, "wb") as fh:
        fh.write(b"WRFC" + struct.pack("<III", 1, 3, 0))
        for o, s in zip(offs, sizes):
            fh.write(struct.pack("<QQ", o, s))
        fh.write(wrf2 + wrfd + trailer)


def read_wrfc(path: str) -> Scene:
    with open(path, "rb") as fh:
        buf = fh.read()
    if buf[:4] != b"WRFC":
        raise RuntimeError("bad magic, not a checkpoint")
    ver, nsec, _ = struct.unpack_from("<III", buf, 4)
    if ver != 1 or nsec != 3:
        raise RuntimeError("unsupported checkpoint")
    table = [struct.unpack_from("<QQ", buf, 16 + 16 * i) for i in range(3)]
    o = table[0][0]
    if buf[o:o + 4] != b"WRF2":
        raise RuntimeError("bad magic, not a gaussian section")
    _, n, _ = struct.unpack_from("<III", buf, o + 4)
    o += 16
    take = lambda cnt: np.frombuffer(buf, "<f4", cnt, o).astype(np.float32)
    cr = take(2 * n).reshape(n, 2); o += 8 * n
    ch = take(3 * n).reshape(n, 3); o += 12 * n
    at = take(n); o += 4 * n
    rs = take(2 * n).reshape(n, 2)
    o = table[1][0]
    if buf[o:o + 4] != b"WRFD":
        raise RuntimeError("bad magic, not a deform section")
    _, cnt, width, bc, bp = struct.unpack_from("<IIIII", buf, o + 4)
    o += 24
    shapes = [struct.unpack_from("<II", buf, o + 8 * i) for i in range(cnt)]
    o += 8 * cnt
    ws, bs = [], []
    for r, c in shapes:
        ws.append(np.frombuffer(buf, "<f4", r * c, o).reshape(r, c).astype(np.float32)); o += 4 * r * c
        bs.append(np.frombuffer(buf, "<f4", r, o).astype(np.float32)); o += 4 * r
    tj = json.loads(buf[table[2][0]:table[2][0] + table[2][1]].decode())
    cfg = tj["config"]
    return Scene(H=tj["grid"]["n_elevation"], W=tj["grid"]["n_azimuth"], center_raw=cr, cholesky=ch,
                 atten_logit=at, response=rs, width=width, bands_c=bc, bands_p=bp, weights=ws, biases=bs,
                 cutoff=float(cfg.get("cutoff_radius", 3.0)), tile=int(cfg.get("tile", 16)),
                 bbox_min=tuple(tj["bbox_min"]), bbox_max=tuple(tj["bbox_max"]),
                 rssi_cal=(tj["rssi_slope"], tj["rssi_intercept"]) if "rssi_slope" in tj and "rssi_intercept" in tj
                 else None)


# ----------------------------------------------------------- synthetic scenes

ROOM_BBOX = ((0.3, 0.3, 0.3), (3.7, 2.7, 2.2))  # default room minus a 0.3 m margin


def _encode(v: np.ndarray, bands: int) -> np.ndarray:
    """deform.cpp:54-70 in float32 for a [rows, count] block."""
    v = v.astype(np.float32)
    out = [v]
    for k in range(bands):
        f = np.float32(math.ldexp(PI, k))
        out += [np.sin(f * v), np.cos(f * v)]
    return np.concatenate(out, axis=1).astype(np.float32)


def _trunk_forward(sc: Scene, x: np.ndarray) -> np.ndarray:
    h = x
    for i in range(TRUNK):
        inp = np.concatenate([h, x], axis=1) if i in SKIP else h
        h = np.maximum(inp @ sc.weights[i].T.astype(np.float64) + sc.biases[i], 0.0)
    return h


def make_scene(n: int, seed: int = 0, H: int = 90, W: int = 360, width: int = 156,
               bands_c: int = 10, bands_p: int = 6, cutoff: float = 3.0, tile: int = 16,
               residual_cells: float = 1.0, fresh_net: bool = False) -> Scene:
    rng = np.random.default_rng(seed)
    cel, caz = (PI / 2.0) / H, (2.0 * PI) / W
    cr = rng.uniform(-2.0, 2.0, size=(n, 2)).astype(np.float32)
    l1 = rng.uniform(0.5, 4.0, size=n) * cel
    l3 = rng.uniform(0.5, 4.0, size=n) * caz
    l2 = rng.uniform(-0.5, 0.5, size=n) * l1
    ch = np.stack([l1, l2, l3], axis=1).astype(np.float32)
    at = rng.uniform(-3.0, 3.0, size=n).astype(np.float32)
    rs = rng.normal(0.0, 0.05, size=(n, 2)).astype(np.float32)
    sc = Scene(H=H, W=W, center_raw=cr, cholesky=ch, atten_logit=at, response=rs, width=width,
               bands_c=bands_c, bands_p=bands_p, cutoff=cutoff, tile=tile,
               bbox_min=ROOM_BBOX[0], bbox_max=ROOM_BBOX[1])
    for r, c in sc.layer_shapes()[:TRUNK]:
        lim = 1.0 / math.sqrt(c)
        sc.weights.append(rng.uniform(-lim, lim, size=(r, c)).astype(np.float32))
        sc.biases.append(np.zeros(r, np.float32))
    for r in (2, 2, 1):
        sc.weights.append(np.zeros((r, width), np.float32))
        sc.biases.append(np.zeros(r, np.float32))
    if fresh_net:
        return sc
    # calibrate the heads on a sample of (Gaussian, position) rows
    m = min(n, 512)
    idx = rng.choice(n, size=m, replace=False)
    el = (np.float32(PI / 4) * (np.tanh(cr[idx, 0]) + np.float32(1))).astype(np.float32)
    az = (np.float32(PI) * (np.tanh(cr[idx, 1]) + np.float32(1))).astype(np.float32)
    pos = rng.uniform(0.0, 1.0, size=(m, 3)).astype(np.float32)
    x = np.concatenate([_encode(np.stack([el, az], 1), bands_c), _encode(pos, bands_p)], axis=1)
    h8 = _trunk_forward(sc, x.astype(np.float64))
    targets = [(8, [residual_cells * cel, residual_cells * caz]), (9, [0.05, 0.05]), (10, [0.05])]
    for li, rms in targets:
        w = rng.uniform(-1.0, 1.0, size=sc.weights[li].shape)
        out = h8 @ w.T
        scale = np.array(rms) / np.maximum(np.sqrt((out ** 2).mean(axis=0)), 1e-30)
        sc.weights[li] = (w * scale[:, None]).astype(np.float32)
    return sc


def random_positions(count: int, seed: int = 0, bbox=ROOM_BBOX) -> np.ndarray:
    rng = np.random.default_rng(seed + 7919)
    lo, hi = np.array(bbox[0]), np.array(bbox[1])
    return (lo + (hi - lo) * rng.uniform(0.0, 1.0, size=(count, 3))).astype(np.float32)


def grid_positions(nx: int, ny: int, nz: int, bbox=ROOM_BBOX) -> np.ndarray:
    """Dense regular TX grid (config 4), x slowest."""
    lo, hi = np.array(bbox[0]), np.array(bbox[1])
    axes = [lo[a] + (hi[a] - lo[a]) * (np.arange(k) + 0.5) / k for a, k in enumerate((nx, ny, nz))]
    g = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)
    return g.astype(np.float32)
