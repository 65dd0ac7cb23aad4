"""Python host for libswr.so, mirroring the reference's render-path API.

Reference C++ API            this module
---------------------------------------------------   -------------------------------------------
train::load_checkpoint(path)         training.hpp:133  load_checkpoint(path, device) -> Checkpoint
train::normalize_position(ck, pos)   training.hpp:149  normalize_position(ck, pos) (batched too)
train::render_at(ck, pos)            training.hpp:154  render_at(ck, pos) / render(ck, positions)
deform::predict_residuals(...)       deform.hpp:106    predict_residuals(ck, pos01) -> Residuals
splat::rasterize(set, res, params)   splat.hpp:152     rasterize(ck, residuals=None)
tasks::pooled_magnitude(spectrum)    tasks.hpp:41      pooled_magnitude(ck, spectra)
tasks::aoa_extract(spectrum)         tasks.hpp:79      aoa_extract(ck, spectra)

Errors follow the reference: size/grid mismatches raise ValueError (the
reference's std::invalid_argument), I/O and format problems RuntimeError.
There is no CPU path: if libswr.so is missing or no sm_100 device is visible,
every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SWR_LIB: an alternative build of the same library (tools/build_variant.py experiments)
LIB_PATH = os.environ.get("SWR_LIB") or os.path.join(_HERE, "libswr.so")

OUT_SPECTRA, OUT_POOLED, OUT_RSSI, OUT_AOA, NO_RESIDUALS = 1, 2, 4, 8, 16
MLP_FP32, MLP_FP16X3, MLP_FP16 = 0, 1, 2

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lib = None


class SwrError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2506_12787_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.swr_last_error.restype = C.c_char_p
        L.swr_launch_count.restype = C.c_int64
        L.swr_launch_count.argtypes = [C.c_void_p]
        L.swr_scene_destroy.argtypes = [C.c_void_p]
        L.swr_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_double]
        L.swr_get_option.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double)]
        L.swr_render.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_render_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        for fn in ("swr_predict_residuals",):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_normalize_positions.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.swr_setup.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_bin.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                              C.c_void_p, C.c_int64, C.c_void_p]
        L.swr_rasterize.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.swr_heads.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_stage_times.argtypes = [C.c_void_p, C.c_void_p]
        L.swr_metrics.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
        L.swr_metrics_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_evaluate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.swr_dataset_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.swr_dataset_close.argtypes = [C.c_void_p]
        L.swr_dataset_get_info.argtypes = [C.c_void_p, C.c_void_p]
        L.swr_dataset_split.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.swr_dataset_read.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.swr_evaluate_dataset.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
        L.swr_group_create.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_group_create_wrfc.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_group_destroy.argtypes = [C.c_void_p]
        L.swr_group_destroy.restype = None
        L.swr_group_size.argtypes = [C.c_void_p, C.c_void_p]
        L.swr_group_context.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_group_render.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32] + [C.c_void_p] * 5
        L.swr_group_render_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint32] + [C.c_void_p] * 6
        L.swr_nccl_unique_id.argtypes = [C.c_void_p]
        L.swr_comm_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_comm_destroy.argtypes = [C.c_void_p]
        L.swr_comm_destroy.restype = None
        L.swr_render_gather.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        L.swr_dataset_get_meta.argtypes = [C.c_void_p, C.c_void_p]
        L.swr_dataset_manifest_json.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p,
                                                C.c_void_p]
        L.swr_dataset_writer_open.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        L.swr_dataset_writer_append.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        L.swr_dataset_writer_render.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        L.swr_dataset_writer_close.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_dataset_save.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.swr_rasterize_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                             C.c_void_p] + [C.c_void_p] * 7
        L.swr_hybrid_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p,
                                      C.c_void_p]
        L.swr_train_config_default.argtypes = [C.c_void_p]
        L.swr_train_config_default.restype = None
        L.swr_trainer_create.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_trainer_destroy.argtypes = [C.c_void_p]
        L.swr_trainer_destroy.restype = None
        L.swr_trainer_run.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_trainer_iteration.argtypes = [C.c_void_p]
        L.swr_trainer_iteration.restype = C.c_int64
        L.swr_trainer_params.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.swr_trainer_gradients.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        L.swr_trainer_save.argtypes = [C.c_void_p, C.c_char_p]
        L.swr_steering_create.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int,
                                          C.POINTER(C.c_void_p)]
        L.swr_steering_destroy.argtypes = [C.c_void_p]
        L.swr_steering_destroy.restype = None
        L.swr_steering_table.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.swr_beam_scan.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.swr_beam_scan_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.swr_beam_scan_targets.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.swr_scene_set_manifest_hash.argtypes = [C.c_void_p, C.c_uint64]
        L.swr_scene_get_info.argtypes = [C.c_void_p, C.c_void_p]
        L.swr_scene_create_wrfc.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.swr_scene_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_float, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().swr_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 4:
        raise ArithmeticError(msg)  # std::domain_error (non-finite metric input)
    raise SwrError(msg)


def _p(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _Info(C.Structure):
    _fields_ = [("n_elevation", C.c_int), ("n_azimuth", C.c_int), ("n", C.c_int), ("width", C.c_int),
                ("bands_center", C.c_int), ("bands_position", C.c_int), ("cutoff_radius", C.c_float),
                ("tile", C.c_int), ("bbox_min", C.c_double * 3), ("bbox_max", C.c_double * 3),
                ("pairs_last", C.c_int64)]


@dataclass
class Residuals:
    """splat::ResidualsT layout per position (splat.hpp:61-72), batched: [B][n][...]."""
    d_center: np.ndarray
    d_response: np.ndarray
    d_atten: np.ndarray


class Checkpoint:
    """A scene (Gaussian set + deform net + raster params + bbox) resident on one B200."""

    def __init__(self, handle, keep=None):
        self._h = C.c_void_p(handle)
        self._keep = keep
        info = _Info()
        _check(lib().swr_scene_get_info(self._h, C.byref(info)))
        self.H, self.W, self.n = info.n_elevation, info.n_azimuth, info.n
        self.width = info.width
        self.cutoff, self.tile = info.cutoff_radius, info.tile
        self.bbox_min, self.bbox_max = tuple(info.bbox_min), tuple(info.bbox_max)
        t = self.tile if self.tile >= 1 else 16
        self.tiles = ((self.H + t - 1) // t) * ((self.W + t - 1) // t)

    @classmethod
    def from_scene(cls, sc, device: int = 0):
        keep = [_f32(sc.center_raw), _f32(sc.cholesky), _f32(sc.atten_logit), _f32(sc.response)]
        lw = lb = None
        if sc.weights:
            ws = [_f32(w) for w in sc.weights]
            bs = [_f32(b) for b in sc.biases]
            keep += ws + bs
            lw = (C.c_void_p * 11)(*[w.ctypes.data for w in ws])
            lb = (C.c_void_p * 11)(*[b.ctypes.data for b in bs])
        bmin = np.array(sc.bbox_min, np.float64)
        bmax = np.array(sc.bbox_max, np.float64)
        h = C.c_void_p()
        _check(lib().swr_scene_create(sc.H, sc.W, sc.n, *[a.ctypes.data for a in keep[:4]], sc.width, sc.bands_c,
                                      sc.bands_p, C.cast(lw, C.c_void_p) if lw else None,
                                      C.cast(lb, C.c_void_p) if lb else None, C.c_float(sc.cutoff), sc.tile,
                                      bmin.ctypes.data, bmax.ctypes.data, device, C.byref(h)))
        ck = cls(h.value)
        if getattr(sc, "rssi_cal", None) is not None:
            ck.set_option("rssi_slope", sc.rssi_cal[0])
            ck.set_option("rssi_intercept", sc.rssi_cal[1])
        return ck

    def set_manifest_hash(self, h: int) -> None:
        """Fingerprint of the dataset this scene was trained on (checkpoint.cpp:133)."""
        _check(lib().swr_scene_set_manifest_hash(self._h, C.c_uint64(h)))

    def close(self):
        if self._h:
            lib().swr_scene_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_option(self, key: str, value: float) -> None:
        _check(lib().swr_set_option(self._h, key.encode(), float(value)))

    def get_option(self, key: str) -> float:
        v = C.c_double(0.0)
        _check(lib().swr_get_option(self._h, key.encode(), C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        return int(lib().swr_launch_count(self._h))

    def pairs_last(self) -> int:
        info = _Info()
        _check(lib().swr_scene_get_info(self._h, C.byref(info)))
        return int(info.pairs_last)

    def stage_times(self):
        out = np.zeros(6, np.float64)
        _check(lib().swr_stage_times(self._h, out.ctypes.data))
        return out


def load_checkpoint(path: str, device: int = 0) -> Checkpoint:
    h = C.c_void_p()
    _check(lib().swr_scene_create_wrfc(path.encode(), device, C.byref(h)))
    return Checkpoint(h.value)


def wrfc_peek(path: str) -> dict:
    """Header + trailer of a WRFC file without a device (swr_wrfc_peek): grid, n,
    net dims, raster params, bbox, and the RSSI calibration of an RSSI model."""
    info = _Info()
    cal = np.zeros(2, np.float64)
    has = C.c_int(0)
    L = lib()
    L.swr_wrfc_peek.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]
    _check(L.swr_wrfc_peek(path.encode(), C.addressof(info), cal.ctypes.data, C.addressof(has)))
    return dict(H=info.n_elevation, W=info.n_azimuth, n=info.n, width=info.width, bands_center=info.bands_center,
                bands_position=info.bands_position, cutoff=info.cutoff_radius, tile=info.tile,
                bbox_min=tuple(info.bbox_min), bbox_max=tuple(info.bbox_max),
                rssi_cal=(float(cal[0]), float(cal[1])) if has.value else None)


def normalize_position(ck: Checkpoint, pos) -> np.ndarray:
    p = _f32(pos).reshape(-1, 3)
    out = np.zeros_like(p)
    _check(lib().swr_normalize_positions(ck.handle, _p(p), p.shape[0], _p(out)))
    return out.reshape(np.shape(pos))


def render(ck: Checkpoint, positions, spectra=True, pooled=True, rssi=False, aoa=True, residuals=True):
    """Batched render_at + heads. Returns dict of numpy arrays."""
    pos = _f32(positions).reshape(-1, 3)
    B = pos.shape[0]
    flags = (OUT_SPECTRA if spectra else 0) | (OUT_POOLED if pooled else 0) | (OUT_RSSI if rssi else 0) \
        | (OUT_AOA if aoa else 0) | (0 if residuals else NO_RESIDUALS)
    out = {}
    sp = np.zeros((B, ck.H, ck.W, 2), np.float32) if spectra else None
    pl = np.zeros(B, np.float64) if pooled else None
    rs = np.zeros(B, np.float64) if rssi else None
    rc = np.zeros((B, 2), np.int32) if aoa else None
    ang = np.zeros((B, 2), np.float64) if aoa else None
    _check(lib().swr_render(ck.handle, _p(pos), B, flags, _p(sp), _p(pl), _p(rs), _p(rc), _p(ang)))
    for k, v in (("spectra", sp), ("pooled", pl), ("rssi", rs), ("aoa_rc", rc), ("aoa_ang", ang)):
        if v is not None:
            out[k] = v
    return out


def render_at(ck: Checkpoint, pos) -> np.ndarray:
    """train::render_at (training.cpp:189-195): one spectrum [H][W][2]."""
    return render(ck, np.asarray(pos, np.float32).reshape(1, 3), pooled=False, aoa=False)["spectra"][0]


def render_device(ck: Checkpoint, d_pos_ptr: int, B: int, flags: int, d_spec=0, d_pooled=0, d_rssi=0, d_aoa_rc=0,
                  d_aoa_ang=0, stream=0) -> None:
    """Stream-ordered render on device pointers (e.g. torch tensors' data_ptr())."""
    _check(lib().swr_render_device(ck.handle, d_pos_ptr, B, flags, d_spec or None, d_pooled or None,
                                   d_rssi or None, d_aoa_rc or None, d_aoa_ang or None, stream or None))


class Group:
    """Multi-GPU render (csrc/group.cpp): one context per device, positions split
    contiguously, outputs gathered to the root (members[0])."""

    def __init__(self, members):
        self.members = list(members)
        arr = (C.c_void_p * len(self.members))(*[m.handle.value for m in self.members])
        h = C.c_void_p()
        _check(lib().swr_group_create(arr, len(self.members), C.byref(h)))
        self._h = h
        self.H, self.W = self.members[0].H, self.members[0].W

    def render(self, positions, spectra=True, pooled=True, rssi=False, aoa=True):
        pos = _f32(positions).reshape(-1, 3)
        B = pos.shape[0]
        flags = (OUT_SPECTRA if spectra else 0) | (OUT_POOLED if pooled else 0) | (OUT_RSSI if rssi else 0) \
            | (OUT_AOA if aoa else 0)
        sp = np.zeros((B, self.H, self.W, 2), np.float32) if spectra else None
        pl = np.zeros(B, np.float64) if pooled else None
        rs = np.zeros(B, np.float64) if rssi else None
        rc = np.zeros((B, 2), np.int32) if aoa else None
        ang = np.zeros((B, 2), np.float64) if aoa else None
        _check(lib().swr_group_render(self._h, _p(pos), B, flags, _p(sp), _p(pl), _p(rs), _p(rc), _p(ang)))
        return {k: v for k, v in (("spectra", sp), ("pooled", pl), ("rssi", rs), ("aoa_rc", rc), ("aoa_ang", ang))
                if v is not None}

    def render_device(self, d_pos_ptr, B, flags, d_spec=0, d_pooled=0, d_rssi=0, d_aoa_rc=0, d_aoa_ang=0, stream=0):
        _check(lib().swr_group_render_device(self._h, d_pos_ptr, B, flags, d_spec or None, d_pooled or None,
                                             d_rssi or None, d_aoa_rc or None, d_aoa_ang or None, stream or None))

    def close(self):
        if getattr(self, "_h", None):
            lib().swr_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().swr_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """Between processes (one per GPU): a communicator over one context;
    render_gather renders this rank's shard and gathers every rank's spectra to rank 0."""

    def __init__(self, ck: Checkpoint, unique_id: bytes, nranks: int, rank: int):
        self.ck, self.nranks, self.rank = ck, nranks, rank
        idb = C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        _check(lib().swr_comm_create(ck.handle, idb, nranks, rank, C.byref(h)))
        self._h = h

    def render_gather(self, d_pos_ptr, counts, flags, d_spec_root=0, d_pooled_root=0, stream=0):
        cnt = np.ascontiguousarray(counts, np.int64)
        _check(lib().swr_render_gather(self._h, d_pos_ptr or None, _p(cnt), flags, d_spec_root or None,
                                       d_pooled_root or None, stream or None))

    def close(self):
        if getattr(self, "_h", None):
            lib().swr_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def predict_residuals(ck: Checkpoint, pos01) -> Residuals:
    p = _f32(pos01).reshape(-1, 3)
    B, n = p.shape[0], ck.n
    dc = np.zeros((B, n, 2), np.float32)
    dr = np.zeros((B, n, 2), np.float32)
    da = np.zeros((B, n), np.float32)
    _check(lib().swr_predict_residuals(ck.handle, _p(p), B, _p(dc), _p(dr), _p(da)))
    return Residuals(dc, dr, da)


def _res_args(res, B_hint=None):
    if res is None:
        return None, None, None, B_hint or 1
    dc = _f32(res.d_center)
    dr = _f32(res.d_response)
    da = _f32(res.d_atten)
    B = dc.shape[0] if dc.ndim == 3 else 1
    return dc, dr, da, B


def setup(ck: Checkpoint, res: Residuals | None = None, B: int = 1):
    dc, dr, da, B = _res_args(res, B)
    n = ck.n
    state = np.zeros((B, n, 11), np.float32)
    rows = np.zeros((B, n, 2), np.int32)
    cols = np.zeros((B, n, 2), np.int32)
    cnt = np.zeros((B, n), np.int32)
    _check(lib().swr_setup(ck.handle, _p(dc), _p(dr), _p(da), B, _p(state), _p(rows), _p(cols), _p(cnt)))
    return dict(state=state, rows=rows, cols=cols, tile_count=cnt)


def bins(ck: Checkpoint, res: Residuals | None = None, B: int = 1):
    """CSR bins per position: list of (tile_offset[tiles+1], tile_prims)."""
    dc, dr, da, B = _res_args(res, B)
    off = np.zeros((B, ck.tiles + 1), np.int32)
    npairs = C.c_int64()
    _check(lib().swr_bin(ck.handle, _p(dc), _p(dr), _p(da), B, _p(off), None, 0, C.byref(npairs)))
    prims = np.zeros(max(npairs.value, 1), np.int32)
    _check(lib().swr_bin(ck.handle, _p(dc), _p(dr), _p(da), B, _p(off), _p(prims), npairs.value, C.byref(npairs)))
    out, at = [], 0
    for b in range(B):
        m = int(off[b, -1])
        out.append((off[b], prims[at:at + m]))
        at += m
    return out


def rasterize(ck: Checkpoint, res: Residuals | None = None, B: int = 1) -> np.ndarray:
    dc, dr, da, B = _res_args(res, B)
    sp = np.zeros((B, ck.H, ck.W, 2), np.float32)
    _check(lib().swr_rasterize(ck.handle, _p(dc), _p(dr), _p(da), B, _p(sp)))
    return sp


# RenderGrads field order and widths (splat.hpp:77-89)
GRAD_FIELDS = (("center_raw", 2), ("cholesky", 3), ("atten_logit", 1), ("response", 2), ("d_center", 2),
               ("d_response", 2), ("d_atten", 1))


def rasterize_backward(ck: Checkpoint, upstream, res: Residuals | None = None) -> dict:
    """splat::rasterize_backward (splat.cpp:494-669) per position: upstream
    dL/dA [B][H][W][2] (+ residuals [B]...) -> the RenderGrads fields, [B][n][w]."""
    up = _f32(upstream).reshape(-1, ck.H, ck.W, 2)
    dc, dr, da, B = _res_args(res, up.shape[0])
    if res is None:
        B = up.shape[0]
    elif B != up.shape[0]:
        raise ValueError("residual and upstream batch sizes differ")
    out = {k: np.zeros((B, ck.n, w) if w > 1 else (B, ck.n), np.float32) for k, w in GRAD_FIELDS}
    _check(lib().swr_rasterize_backward(ck.handle, _p(dc), _p(dr), _p(da), B, _p(up),
                                        *[_p(out[k]) for k, _ in GRAD_FIELDS]))
    return out


def hybrid_loss(ck: Checkpoint, pred, target, lambda1: float = 0.8, grad: bool = True):
    """train::hybrid_loss (training.cpp:62-106) per pair: (terms [B][3] =
    (loss, l1_term, ssim_term), dLoss/dprediction [B][H][W][2] or None)."""
    a = _f32(pred).reshape(-1, ck.H, ck.W, 2)
    b = _f32(target).reshape(-1, ck.H, ck.W, 2)
    if a.shape != b.shape:
        raise ValueError("spectrum shape mismatch")
    B = a.shape[0]
    terms = np.zeros((B, 3), np.float64)
    g = np.zeros_like(a) if grad else None
    _check(lib().swr_hybrid_loss(ck.handle, _p(a), _p(b), B, float(lambda1), _p(terms), _p(g)))
    return terms, g


def heads(ck: Checkpoint, spectra):
    sp = _f32(spectra).reshape(-1, ck.H, ck.W, 2)
    B = sp.shape[0]
    pooled = np.zeros(B, np.float64)
    rc = np.zeros((B, 2), np.int32)
    ang = np.zeros((B, 2), np.float64)
    _check(lib().swr_heads(ck.handle, _p(sp), B, _p(pooled), _p(rc), _p(ang)))
    return pooled, rc, ang


def pooled_magnitude(ck: Checkpoint, spectra) -> np.ndarray:
    return heads(ck, spectra)[0]


def aoa_extract(ck: Checkpoint, spectra):
    _, rc, ang = heads(ck, spectra)
    return rc, ang


def metrics(ck: Checkpoint, pred, target, peak: float = 1.0, ssim: bool = True):
    """psnr / ssim / l1 per spectrum pair (spectrum.cpp:145-250), [B] each."""
    a = _f32(pred).reshape(-1, ck.H, ck.W, 2)
    b = _f32(target).reshape(-1, ck.H, ck.W, 2)
    if a.shape != b.shape:
        raise ValueError("spectrum shape mismatch")
    B = a.shape[0]
    out = {k: np.zeros(B, np.float64) for k in ("psnr", "ssim", "l1")}
    _check(lib().swr_metrics(ck.handle, _p(a), _p(b), B, float(peak), _p(out["psnr"]),
                             _p(out["ssim"]) if ssim else None, _p(out["l1"])))
    if not ssim:
        out.pop("ssim")
    return out


def evaluate(ck: Checkpoint, positions, targets, peak: float = 1.0):
    """train::evaluate (training.cpp:380-406) on a batch: render + score on the device."""
    pos = _f32(positions).reshape(-1, 3)
    t = _f32(targets).reshape(-1, ck.H, ck.W, 2)
    if t.shape[0] != pos.shape[0]:
        raise ValueError("one target spectrum per position")
    B = pos.shape[0]
    out = {k: np.zeros(B, np.float64) for k in ("psnr", "ssim", "l1")}
    _check(lib().swr_evaluate(ck.handle, _p(pos), _p(t), B, float(peak), _p(out["psnr"]), _p(out["ssim"]),
                              _p(out["l1"])))
    return out


class _DsInfo(C.Structure):
    _fields_ = [("n_elevation", C.c_int), ("n_azimuth", C.c_int), ("samples", C.c_int64), ("n_train", C.c_int64),
                ("n_test", C.c_int64), ("n_excluded", C.c_int64), ("manifest_hash", C.c_uint64),
                ("normalization", C.c_double), ("bbox_min", C.c_double * 3), ("bbox_max", C.c_double * 3)]


class DatasetMeta(C.Structure):
    """swr_dataset_meta: the manifest fields of wavesim.hpp:125-139's Dataset."""
    _fields_ = [("n_elevation", C.c_int32), ("n_azimuth", C.c_int32), ("mode", C.c_char_p),
                ("k_elements", C.c_int32), ("spacing", C.c_double), ("wavelength", C.c_double),
                ("room", C.c_double * 3), ("reflectivity", C.c_double), ("max_bounces", C.c_int32),
                ("fixed_node", C.c_double * 3), ("normalization", C.c_double), ("seed", C.c_uint64),
                ("train_indices", C.c_void_p), ("test_indices", C.c_void_p), ("excluded_indices", C.c_void_p),
                ("n_train", C.c_int64), ("n_test", C.c_int64), ("n_excluded", C.c_int64),
                ("bbox_min", C.c_double * 3), ("bbox_max", C.c_double * 3),
                ("rssi_dbm", C.c_void_p), ("n_rssi", C.c_int64)]

    @staticmethod
    def build(H, W, *, mode="tx_moving", k_elements=16, spacing=0.0625, wavelength=0.125,
              room=(4.0, 3.0, 2.5), reflectivity=0.6, max_bounces=1, fixed_node=(2.0, 1.5, 1.25),
              normalization=1.0, seed=0, train=(), test=(), excluded=(), bbox_min=(0, 0, 0), bbox_max=(1, 1, 1),
              rssi_dbm=()):
        m = DatasetMeta()
        m.n_elevation, m.n_azimuth = H, W
        m._keep = [mode.encode()] + [np.ascontiguousarray(v, np.int32) for v in (train, test, excluded)] + \
                  [np.ascontiguousarray(rssi_dbm, np.float64)]
        m.mode = m._keep[0]
        m.k_elements, m.spacing, m.wavelength = k_elements, spacing, wavelength
        m.room[:] = list(room)
        m.reflectivity, m.max_bounces = reflectivity, max_bounces
        m.fixed_node[:] = list(fixed_node)
        m.normalization, m.seed = normalization, seed
        (tr, te, ex, rs) = m._keep[1:]
        m.train_indices, m.test_indices, m.excluded_indices = _p(tr), _p(te), _p(ex)
        m.n_train, m.n_test, m.n_excluded = len(tr), len(te), len(ex)
        m.bbox_min[:] = list(bbox_min)
        m.bbox_max[:] = list(bbox_max)
        m.rssi_dbm, m.n_rssi = _p(rs), len(rs)
        return m

    def manifest(self, sample_count: int):
        """(manifest.json bytes exactly as manifest_json writes them, FNV-1a 64 hash)"""
        n, h = C.c_size_t(), C.c_uint64()
        _check(lib().swr_dataset_manifest_json(C.byref(self), sample_count, None, 0, C.byref(n), C.byref(h)))
        buf = C.create_string_buffer(n.value)
        _check(lib().swr_dataset_manifest_json(C.byref(self), sample_count, buf, n.value, C.byref(n), C.byref(h)))
        return buf.raw[:n.value], h.value


class DatasetWriter:
    """save_dataset (dataset.cpp:183-203) as a stream: append host records or render
    positions on the GPU; close(meta) writes manifest.json and returns its hash."""

    def __init__(self, path: str, H: int, W: int):
        h = C.c_void_p()
        _check(lib().swr_dataset_writer_open(path.encode(), H, W, C.byref(h)))
        self._h = h

    def append(self, pos, spectra):
        pos = np.ascontiguousarray(pos, np.float32)
        spectra = np.ascontiguousarray(spectra, np.float32)
        _check(lib().swr_dataset_writer_append(self._h, _p(pos), _p(spectra), len(pos)))

    def render(self, ck: "Checkpoint", pos_m):
        pos_m = np.ascontiguousarray(pos_m, np.float32)
        _check(lib().swr_dataset_writer_render(self._h, ck.handle, _p(pos_m), len(pos_m)))

    def close(self, meta: DatasetMeta) -> int:
        h = C.c_uint64()
        w, self._h = self._h, None
        _check(lib().swr_dataset_writer_close(w, C.byref(meta), C.byref(h)))
        return h.value


def save_dataset(path: str, meta: DatasetMeta, pos, spectra) -> int:
    pos = np.ascontiguousarray(pos, np.float32)
    spectra = np.ascontiguousarray(spectra, np.float32)
    h = C.c_uint64()
    _check(lib().swr_dataset_save(path.encode(), C.byref(meta), _p(pos), _p(spectra), len(pos), C.byref(h)))
    return h.value


class Dataset:
    """manifest.json + spectra.bin reader (load_dataset, dataset.cpp:205-258), records on demand."""

    TRAIN, TEST, ALL = 0, 1, 2

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(lib().swr_dataset_open(path.encode(), C.byref(h)))
        self._h = h
        info = _DsInfo()
        _check(lib().swr_dataset_get_info(self._h, C.byref(info)))
        self.H, self.W, self.samples = info.n_elevation, info.n_azimuth, info.samples
        self.manifest_hash = info.manifest_hash
        self.bbox = np.array(list(info.bbox_min) + list(info.bbox_max))
        self.normalization = info.normalization

    def meta(self) -> DatasetMeta:
        """the full manifest (pointers into this reader's storage: keep it open)"""
        m = DatasetMeta()
        _check(lib().swr_dataset_get_meta(self._h, C.byref(m)))
        m._owner = self
        return m

    def split(self, which: int) -> np.ndarray:
        n = C.c_int64()
        _check(lib().swr_dataset_split(self._h, which, None, C.byref(n)))
        idx = np.zeros(n.value, np.int32)
        _check(lib().swr_dataset_split(self._h, which, _p(idx), C.byref(n)))
        return idx

    def read(self, indices=None, count=None):
        idx = None if indices is None else np.ascontiguousarray(indices, np.int32)
        n = len(idx) if idx is not None else (self.samples if count is None else count)
        pos = np.zeros((n, 3), np.float32)
        spec = np.zeros((n, self.H, self.W, 2), np.float32)
        _check(lib().swr_dataset_read(self._h, _p(idx), n, _p(pos), _p(spec)))
        return pos, spec

    def close(self):
        if self._h:
            lib().swr_dataset_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def evaluate_dataset(ck: Checkpoint, ds: Dataset, split: int):
    """train::evaluate (training.cpp:380-406): per sample of the split (ids, psnr, ssim, l1)."""
    n = len(ds.split(split))
    out = {"sample_id": np.zeros(n, np.int32), "psnr": np.zeros(n), "ssim": np.zeros(n), "l1": np.zeros(n)}
    _check(lib().swr_evaluate_dataset(ck.handle, ds._h, split, _p(out["sample_id"]), _p(out["psnr"]),
                                      _p(out["ssim"]), _p(out["l1"])))
    return out


# ---------------------------------------------------------------- training

class TrainConfig(C.Structure):
    """train::TrainConfig (training.hpp:96-112); defaults are the reference's."""
    _fields_ = [("primitives", C.c_int32), ("bands_center", C.c_int32), ("bands_position", C.c_int32),
                ("width", C.c_int32), ("cutoff_radius", C.c_float), ("tile", C.c_int32),
                ("lr_gaussian", C.c_double), ("lr_mlp", C.c_double), ("lambda1", C.c_double),
                ("coarse_iters", C.c_int64), ("fine_iters", C.c_int64), ("anneal_scale", C.c_double),
                ("anneal_threshold", C.c_int64), ("seed", C.c_uint64)]

    def __init__(self, **kw):
        super().__init__()
        lib().swr_train_config_default(C.byref(self))
        for k, v in kw.items():
            if not hasattr(self, k):
                raise TypeError(f"unknown TrainConfig field {k}")
            setattr(self, k, v)


def _layer_shapes(width, bands_c, bands_p):
    D = 2 * (2 * bands_c + 1) + 3 * (2 * bands_p + 1)
    cols = [D if i == 0 else (width + D if i in (2, 4, 6) else width) for i in range(8)]
    return [(width, c) for c in cols] + [(2, width), (2, width), (1, width)]


class Trainer:
    """train::train (training.cpp:198-376) on one B200: create (fresh or resume),
    run iterations of the coarse/fine schedule, read / save the parameters."""

    def __init__(self, cfg: TrainConfig, ds: Dataset, resume: str | None = None, device: int = 0):
        self.cfg = cfg
        h = C.c_void_p()
        _check(lib().swr_trainer_create(C.byref(cfg), ds._h, resume.encode() if resume else None, device,
                                        C.byref(h)))
        self._h = h
        self.H, self.W = ds.H, ds.W
        self.n = None

    @property
    def iteration(self) -> int:
        return int(lib().swr_trainer_iteration(self._h))

    def run(self, iters: int | None = None):
        """Run up to `iters` iterations (default: the rest of the schedule).
        Returns (log [k][3] = loss, l1_term, ssim_term; device ms)."""
        total = self.cfg.coarse_iters + self.cfg.fine_iters
        k = total - self.iteration if iters is None else int(iters)
        k = max(k, 0)
        log = np.zeros((k, 3), np.float64)
        done = C.c_int64()
        ms = C.c_double()
        _check(lib().swr_trainer_run(self._h, k, _p(log), C.byref(done), C.byref(ms)))
        return log[:done.value], ms.value

    def params(self) -> dict:
        n = self._count()
        out = {"center_raw": np.zeros((n, 2), np.float32), "cholesky": np.zeros((n, 3), np.float32),
               "atten_logit": np.zeros(n, np.float32), "response": np.zeros((n, 2), np.float32)}
        shapes = _layer_shapes(self.cfg.width, self.cfg.bands_center, self.cfg.bands_position)
        out["weights"] = [np.zeros(s, np.float32) for s in shapes]
        out["biases"] = [np.zeros(s[0], np.float32) for s in shapes]
        pw = (C.c_void_p * 11)(*[w.ctypes.data for w in out["weights"]])
        pb = (C.c_void_p * 11)(*[b.ctypes.data for b in out["biases"]])
        _check(lib().swr_trainer_params(self._h, _p(out["center_raw"]), _p(out["cholesky"]), _p(out["atten_logit"]),
                                        _p(out["response"]), pw, pb))
        return out

    def _count(self) -> int:
        # the Gaussian count: cfg.primitives (a resumed checkpoint must carry the same config)
        if self.n is None:
            self.n = int(self.cfg.primitives)
        return self.n

    def gradients(self, sample: int, pos01=None) -> dict:
        """One forward/backward at the current parameters (no step). pos01 given:
        the fine-stage chain incl. DeformGrads; else the coarse chain."""
        n = self._count()
        g = {k: np.zeros((n, w) if w > 1 else n, np.float32) for k, w in GRAD_FIELDS}
        terms = np.zeros(3)
        rg = (C.c_void_p * 7)(*[g[k].ctypes.data for k, _ in GRAD_FIELDS])
        shapes = _layer_shapes(self.cfg.width, self.cfg.bands_center, self.cfg.bands_position)
        gw = [np.zeros(s, np.float32) for s in shapes]
        gb = [np.zeros(s[0], np.float32) for s in shapes]
        pos = None if pos01 is None else _f32(pos01).reshape(3)
        _check(lib().swr_trainer_gradients(self._h, _p(pos), int(sample), _p(terms), rg,
                                           (C.c_void_p * 11)(*[w.ctypes.data for w in gw]),
                                           (C.c_void_p * 11)(*[b.ctypes.data for b in gb])))
        g["terms"] = terms
        if pos is not None:
            g["layer_w"], g["layer_b"] = gw, gb
        return g

    def save(self, path: str) -> None:
        _check(lib().swr_trainer_save(self._h, path.encode()))

    def close(self):
        if getattr(self, "_h", None):
            lib().swr_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def train(ds: Dataset, cfg: TrainConfig, resume: str | None = None, device: int = 0):
    """train::train: the whole schedule; returns (trainer, log [iters][3])."""
    tr = Trainer(cfg, ds, resume, device)
    log, _ = tr.run()
    return tr, log


# ---------------------------------------------------------------- beam scan

class Steering:
    """sim::SteeringTable on one B200 (wavesim.cpp:183-211) + batched beam_scan
    (wavesim.cpp:213-252) and generate_dataset's targets (dataset.cpp:86-124)."""

    def __init__(self, H: int, W: int, k_elements: int = 16, spacing: float = 0.0625, wavelength: float = 0.125,
                 device: int = 0):
        h = C.c_void_p()
        _check(lib().swr_steering_create(int(k_elements), float(spacing), float(wavelength), int(H), int(W), device,
                                         C.byref(h)))
        self._h = h
        self.H, self.W, self.k = H, W, k_elements

    def table(self):
        wr = np.zeros((self.H * self.W, self.k), np.float64)
        wi = np.zeros_like(wr)
        _check(lib().swr_steering_table(self._h, _p(wr), _p(wi)))
        return wr, wi

    def scan(self, channels) -> np.ndarray:
        """channels [B][K] complex -> spectra [B][H][W][2] float64."""
        ch = np.ascontiguousarray(np.asarray(channels, np.complex128).reshape(-1, self.k))
        B = ch.shape[0]
        out = np.zeros((B, self.H, self.W, 2), np.float64)
        _check(lib().swr_beam_scan(self._h, _p(ch.view(np.float64)), B, _p(out)))
        return out

    def targets(self, channels):
        """Dataset targets [B][H][W][2] float32 (|A| / max|A|, imaginary 0) and the normalization."""
        ch = np.ascontiguousarray(np.asarray(channels, np.complex128).reshape(-1, self.k))
        B = ch.shape[0]
        out = np.zeros((B, self.H, self.W, 2), np.float32)
        norm = C.c_double()
        _check(lib().swr_beam_scan_targets(self._h, _p(ch.view(np.float64)), B, _p(out), C.byref(norm)))
        return out, norm.value

    def close(self):
        if getattr(self, "_h", None):
            lib().swr_steering_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
