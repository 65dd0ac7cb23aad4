"""ctypes access to the CPU checkers. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
`--impl reference` arm) may import this module. It never backs the product.

* `Port`      -> oracle/liboracle.so, the plain-C restatement (swr_oracle.c)
* `Reference` -> oracle/_ref/libwrfref.so (or _nofma), the reference library
                 compiled from /root/reference sources (oracle/Makefile)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwrfref.so")
REF_NOFMA_SO = os.path.join(HERE, "_ref", "libwrfref_nofma.so")
REF_BLAS_SO = os.path.join(HERE, "_ref", "libwrfref_blas.so")
REF_BLAS_V4_SO = os.path.join(HERE, "_ref", "libwrfref_blas_v4.so")


def host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            flags = next((ln for ln in fh if ln.startswith("flags")), "")
        return all(f in flags.split() for f in ("avx512f", "avx512bw", "avx512vl", "avx512dq"))
    except OSError:
        return False


def blas_library() -> str | None:
    """numpy's bundled OpenBLAS (ILP64 CBLAS symbols scipy_cblas_*64_)."""
    import glob
    d = os.path.join(os.path.dirname(os.path.dirname(np.__file__)), "numpy.libs")
    hits = sorted(glob.glob(os.path.join(d, "libscipy_openblas64_*.so")))
    return hits[0] if hits else None


def reference_so(variant: str = "loop") -> str:
    """loop: the restated GEMM loop (-march=x86-64-v3); blas: real SGEMM, the
    x86-64-v4 build on AVX-512 hosts; nofma: -ffp-contract=off."""
    if variant == "nofma":
        return REF_NOFMA_SO
    if variant == "blas":
        return REF_BLAS_V4_SO if host_has_avx512() and os.path.exists(REF_BLAS_V4_SO) else REF_BLAS_SO
    return REF_SO

_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """Compile the checkers (liboracle.so always; _ref only where the reference sources exist)."""
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/src") else [])
    subprocess.run(["make", "-s", "-j4", "-C", HERE] + targets, check=True)


def _f(a):
    return a.ctypes.data_as(_fp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _SoSet(C.Structure):
    _fields_ = [("H", C.c_int), ("W", C.c_int), ("n", C.c_int), ("center_raw", _fp),
                ("cholesky", _fp), ("atten_logit", _fp), ("response", _fp)]


class _SoNet(C.Structure):
    _fields_ = [("width", C.c_int), ("bands_c", C.c_int), ("bands_p", C.c_int),
                ("w", _fp * 11), ("b", _fp * 11)]


def _split_res(res):
    if res is None:
        return None, None, None
    dc, dr, da = res
    return _c32(dc), _c32(dr), _c32(da)


class Port:
    """The plain-C restatement (swr_oracle.c)."""

    def __init__(self, scene):
        self.lib = C.CDLL(PORT_SO)
        L = self.lib
        L.so_prepare.restype = C.c_int64
        L.so_pooled.restype = C.c_double
        self.sc = scene
        self._keep = [_c32(scene.center_raw), _c32(scene.cholesky), _c32(scene.atten_logit),
                      _c32(scene.response)]
        self.set = _SoSet(scene.H, scene.W, scene.n, *[_f(a) for a in self._keep])
        self._w = [_c32(w) for w in scene.weights]
        self._b = [_c32(b) for b in scene.biases]
        if self._w:
            self.net = _SoNet(scene.width, scene.bands_c, scene.bands_p,
                              (_fp * 11)(*[_f(w) for w in self._w]), (_fp * 11)(*[_f(b) for b in self._b]))

    def normalize(self, pos_m):
        out = np.zeros(3, np.float32)
        bmin = np.array(self.sc.bbox_min, np.float64)
        bmax = np.array(self.sc.bbox_max, np.float64)
        self.lib.so_normalize_position(_d(bmin), _d(bmax), _f(_c32(pos_m)), _f(out))
        return out

    def predict(self, pos01, precise=False):
        n = self.sc.n
        dc, dr, da = np.zeros((n, 2), np.float32), np.zeros((n, 2), np.float32), np.zeros(n, np.float32)
        rc = self.lib.so_predict(C.byref(self.net), C.byref(self.set), _f(_c32(pos01)), int(precise),
                                 _f(dc), _f(dr), _f(da))
        if rc:
            raise RuntimeError(f"so_predict failed ({rc})")
        return dc, dr, da

    def prepare(self, res=None):
        sc = self.sc
        dc, dr, da = _split_res(res)
        n = sc.n
        tiles = ((sc.H + sc.tile - 1) // sc.tile) * ((sc.W + sc.tile - 1) // sc.tile)
        state = np.zeros((n, 11), np.float32)
        rows = np.zeros((n, 2), np.int32)
        cols = np.zeros((n, 2), np.int32)
        off = np.zeros(tiles + 1, np.int32)
        pairs = self.lib.so_prepare(C.byref(self.set), _f(dc), _f(dr), _f(da), C.c_float(sc.cutoff), sc.tile,
                                    _f(state), _i(rows), _i(cols), _i(off), None, C.c_int64(0))
        prims = np.zeros(max(pairs, 1), np.int32)
        self.lib.so_prepare(C.byref(self.set), _f(dc), _f(dr), _f(da), C.c_float(sc.cutoff), sc.tile,
                            _f(state), _i(rows), _i(cols), _i(off), _i(prims), C.c_int64(pairs))
        return dict(state=state, rows=rows, cols=cols, tile_offset=off, tile_prims=prims[:pairs])

    def rasterize(self, res=None, precise=True):
        sc = self.sc
        dc, dr, da = _split_res(res)
        out = np.zeros((sc.H, sc.W, 2), np.float32)
        self.lib.so_rasterize(C.byref(self.set), _f(dc), _f(dr), _f(da), C.c_float(sc.cutoff), sc.tile,
                              int(precise), _f(out))
        return out

    def render(self, pos_m, precise=True):
        res = self.predict(self.normalize(pos_m), precise=precise)
        return self.rasterize(res, precise=precise), res

    def aoa(self, spec):
        H, W = spec.shape[0], spec.shape[1]
        r, c, el, az = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        self.lib.so_aoa(_f(_c32(spec)), H, W, C.byref(r), C.byref(c), C.byref(el), C.byref(az))
        return r.value, c.value, el.value, az.value

    def pooled(self, spec):
        return self.lib.so_pooled(_f(_c32(spec)), spec.shape[0] * spec.shape[1])

    def metrics(self, pred, target, peak=1.0, ssim=True):
        """(psnr, ssim, l1) of one spectrum pair (spectrum.cpp:145-250); ssim None if not asked."""
        pred, target = _c32(pred), _c32(target)
        out = [C.c_double(), C.c_double(), C.c_double()]
        rc = self.lib.so_metrics(_f(pred), _f(target), pred.shape[0], pred.shape[1], C.c_double(peak),
                                 C.byref(out[0]), C.byref(out[1]) if ssim else None, C.byref(out[2]))
        if rc == 1:
            raise ArithmeticError("spectrum contains a non-finite value")
        if rc == 2:
            raise ValueError("grid too small for the 11x11 SSIM window")
        return out[0].value, (out[1].value if ssim else None), out[2].value


class Reference:
    """The reference library built from /root/reference sources (oracle/_ref)."""

    def __init__(self, scene=None, path=None, nofma=False, handle=None, variant=None):
        variant = variant or ("nofma" if nofma else "loop")
        so = reference_so(variant)
        if not os.path.exists(so):
            raise FileNotFoundError(f"{so} missing: run `make -C oracle ref` where /root/reference exists")
        if variant == "blas":
            lib = blas_library()
            if lib is None:
                raise FileNotFoundError("numpy's OpenBLAS not found (the blas reference variant needs it)")
            os.environ["WREF_BLAS_LIB"] = lib
        self.variant, self.so = variant, so
        self.lib = L = C.CDLL(so)
        L.wref_ck_load.restype = C.c_void_p
        L.wref_ck_create.restype = C.c_void_p
        L.wref_ck_init_random.restype = C.c_void_p
        L.wref_last_error.restype = C.c_char_p
        L.wref_pooled.restype = C.c_double
        L.wref_kernel_weight.restype = C.c_float
        for fn in ("wref_ck_save", "wref_ck_free", "wref_ck_info", "wref_normalize", "wref_predict",
                   "wref_rasterize", "wref_render_at", "wref_render_batch", "wref_ck_arrays"):
            getattr(L, fn).argtypes = None
        self.sc = scene
        if handle is not None:
            self.h = handle
        elif path is not None:
            self.h = L.wref_ck_load(path.encode())
        else:
            sc = scene
            self._keep = [_c32(sc.center_raw), _c32(sc.cholesky), _c32(sc.atten_logit), _c32(sc.response)]
            lw = lb = None
            if sc.weights:
                self._w = [_c32(w) for w in sc.weights]
                self._b = [_c32(b) for b in sc.biases]
                lw = (_fp * 11)(*[_f(w) for w in self._w])
                lb = (_fp * 11)(*[_f(b) for b in self._b])
            bmin = np.array(sc.bbox_min, np.float64)
            bmax = np.array(sc.bbox_max, np.float64)
            self.h = L.wref_ck_create(sc.H, sc.W, sc.n, *[_f(a) for a in self._keep], sc.width, sc.bands_c,
                                      sc.bands_p, lw, lb, C.c_float(sc.cutoff), sc.tile, _d(bmin), _d(bmax))
        if not self.h:
            raise RuntimeError(self.lib.wref_last_error().decode())
        self.h = C.c_void_p(self.h)
        if self.sc is None:
            self.sc = self._scene_from_handle()

    def _scene_from_handle(self):
        from paper_2506_12787_b200.scene import Scene
        ints = np.zeros(6, np.int32)
        cut = C.c_float()
        bbox = np.zeros(6, np.float64)
        bp = self.lib.wref_ck_info(self.h, _i(ints), C.byref(cut), _d(bbox))
        H, W, n, width, bc, tile = map(int, ints)
        sc = Scene(H=H, W=W, center_raw=np.zeros((n, 2), np.float32), cholesky=np.zeros((n, 3), np.float32),
                   atten_logit=np.zeros(n, np.float32), response=np.zeros((n, 2), np.float32),
                   width=width, bands_c=bc, bands_p=bp, cutoff=cut.value, tile=tile,
                   bbox_min=tuple(bbox[:3]), bbox_max=tuple(bbox[3:]))
        sc.weights = [np.zeros(s, np.float32) for s in sc.layer_shapes()]
        sc.biases = [np.zeros(s[0], np.float32) for s in sc.layer_shapes()]
        self.lib.wref_ck_arrays(self.h, _f(sc.center_raw), _f(sc.cholesky), _f(sc.atten_logit),
                                _f(sc.response), (_fp * 11)(*[_f(w) for w in sc.weights]),
                                (_fp * 11)(*[_f(b) for b in sc.biases]))
        return sc

    def __del__(self):
        try:
            self.lib.wref_ck_free(self.h)
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.lib.wref_last_error().decode())

    def set_threads(self, n):
        self.lib.wref_set_threads(int(n))

    def save(self, path):
        self._check(self.lib.wref_ck_save(self.h, path.encode()))

    def save_rssi_model(self, path, slope, intercept):
        """tasks::save_rssi_model (tasks.cpp:131-137)."""
        self._check(self.lib.wref_save_rssi_model(self.h, path.encode(), C.c_double(slope), C.c_double(intercept)))

    def load_rssi_model(self, path):
        """tasks::load_rssi_model (tasks.cpp:139-150) -> (slope, intercept)."""
        out = np.zeros(2, np.float64)
        self._check(self.lib.wref_load_rssi_model(path.encode(), _d(out)))
        return float(out[0]), float(out[1])

    def normalize(self, pos_m):
        out = np.zeros(3, np.float32)
        self._check(self.lib.wref_normalize(self.h, _f(_c32(pos_m)), _f(out)))
        return out

    def predict(self, pos01):
        n = self.sc.n
        dc, dr, da = np.zeros((n, 2), np.float32), np.zeros((n, 2), np.float32), np.zeros(n, np.float32)
        self._check(self.lib.wref_predict(self.h, _f(_c32(pos01)), _f(dc), _f(dr), _f(da)))
        return dc, dr, da

    def rasterize(self, res=None, workspace=False):
        sc = self.sc
        n = sc.n
        dc, dr, da = _split_res(res)
        tiles = ((sc.H + sc.tile - 1) // sc.tile) * ((sc.W + sc.tile - 1) // sc.tile)
        out = np.zeros((sc.H, sc.W, 2), np.float32)
        if not workspace:
            self._check(self.lib.wref_rasterize(self.h, _f(dc), _f(dr), _f(da), _f(out), None, None, None,
                                                None, None, C.c_longlong(0), None))
            return out
        state = np.zeros((n, 11), np.float32)
        rows = np.zeros((n, 2), np.int32)
        cols = np.zeros((n, 2), np.int32)
        off = np.zeros(tiles + 1, np.int32)
        npairs = C.c_longlong()
        self._check(self.lib.wref_rasterize(self.h, _f(dc), _f(dr), _f(da), _f(out), _f(state), _i(rows),
                                            _i(cols), _i(off), None, C.c_longlong(0), C.byref(npairs)))
        prims = np.zeros(max(npairs.value, 1), np.int32)
        self._check(self.lib.wref_rasterize(self.h, _f(dc), _f(dr), _f(da), None, None, None, None, None,
                                            _i(prims), C.c_longlong(npairs.value), None))
        return out, dict(state=state, rows=rows, cols=cols, tile_offset=off, tile_prims=prims[:npairs.value])

    def render_at(self, pos_m):
        out = np.zeros((self.sc.H, self.sc.W, 2), np.float32)
        self._check(self.lib.wref_render_at(self.h, _f(_c32(pos_m)), _f(out)))
        return out

    def render_batch(self, pos_m, mode=1, spectra=True):
        pos = _c32(pos_m).reshape(-1, 3)
        B = pos.shape[0]
        sp = np.zeros((B, self.sc.H, self.sc.W, 2), np.float32) if spectra else None
        pooled = np.zeros(B, np.float64)
        rc = np.zeros((B, 2), np.int32)
        ang = np.zeros((B, 2), np.float64)
        self._check(self.lib.wref_render_batch(self.h, B, _f(pos), _f(sp), _d(pooled), _i(rc), _d(ang), mode))
        return sp, pooled, rc, ang

    def aoa(self, spec):
        H, W = spec.shape[0], spec.shape[1]
        r, c, el, az = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        self._check(self.lib.wref_aoa(_f(_c32(spec)), H, W, C.byref(r), C.byref(c), C.byref(el), C.byref(az)))
        return r.value, c.value, el.value, az.value

    def pooled(self, spec):
        return self.lib.wref_pooled(_f(_c32(spec)), spec.shape[0], spec.shape[1])

    def set_dataset(self, manifest_hash, bbox6):
        """Bind the checkpoint to a dataset: its manifest hash and normalisation box."""
        b = np.asarray(bbox6, np.float64)
        self.lib.wref_ck_set_dataset(self.h, C.c_uint64(manifest_hash), _d(b))

    def evaluate(self, dataset_dir, split):
        """train::evaluate (training.cpp:380-406): rows [n][4] = (sample id, psnr, ssim, l1)."""
        L = self.lib
        L.wref_evaluate.restype = C.c_longlong
        rows = np.zeros((65536, 4))
        n = L.wref_evaluate(self.h, dataset_dir.encode(), int(split), _d(rows), C.c_longlong(len(rows)))
        if n == -2:
            raise RuntimeError("hash mismatch: " + L.wref_last_error().decode())
        if n < 0:
            raise RuntimeError(L.wref_last_error().decode())
        return rows[:n]

    def metrics(self, pred, target, peak=1.0):
        """(psnr, ssim, l1) through the reference's own psnr / ssim / l1."""
        pred, target = _c32(pred), _c32(target)
        out = np.zeros(3)
        rc = self.lib.wref_metrics(_f(pred), _f(target), pred.shape[0], pred.shape[1], C.c_double(peak), _d(out))
        if rc == 1:
            raise ArithmeticError("spectrum contains a non-finite value")
        if rc == 2:
            raise ValueError("grid too small for the 11x11 SSIM window")
        return tuple(out)

    def rasterize_backward(self, upstream, res=None):
        """splat::rasterize_backward -> dict of the seven RenderGrads fields."""
        n = self.sc.n
        dc, dr, da = _split_res(res)
        widths = (2, 3, 1, 2, 2, 2, 1)
        flat = np.zeros(n * sum(widths), np.float32)
        self._check(self.lib.wref_rasterize_backward(self.h, _f(dc), _f(dr), _f(da), _f(_c32(upstream)), _f(flat)))
        out, at = {}, 0
        names = ("center_raw", "cholesky", "atten_logit", "response", "d_center", "d_response", "d_atten")
        for k, w in zip(names, widths):
            v = flat[at:at + n * w]
            out[k] = v.reshape(n, w) if w > 1 else v.copy()
            at += n * w
        return out

    def hybrid_loss(self, pred, target, lambda1, grad=True):
        pred, target = _c32(pred), _c32(target)
        terms = np.zeros(3)
        g = np.zeros_like(pred) if grad else None
        rc = self.lib.wref_hybrid_loss(_f(pred), _f(target), pred.shape[0], pred.shape[1], C.c_double(lambda1),
                                       _d(terms), _f(g) if grad else None)
        if rc:
            raise ArithmeticError("hybrid loss: non-finite input or loss")
        return terms, g

    def train(self, dataset_dir, cfg, log_path=None, resume=None):
        """train::train(load_dataset(dir), cfg, log_path, resume) -> a new Reference.
        cfg: any object with the TrainConfig fields."""
        L = self.lib
        L.wref_train.restype = C.c_void_p
        ints = (C.c_int * 5)(cfg.primitives, cfg.bands_center, cfg.bands_position, cfg.width, cfg.tile)
        dbl = (C.c_double * 5)(cfg.cutoff_radius, cfg.lr_gaussian, cfg.lr_mlp, cfg.lambda1, cfg.anneal_scale)
        ll = (C.c_longlong * 3)(cfg.coarse_iters, cfg.fine_iters, cfg.anneal_threshold)
        kind = C.c_int()
        h = L.wref_train(dataset_dir.encode(), ints, dbl, ll, C.c_ulonglong(cfg.seed),
                         log_path.encode() if log_path else None, resume.h if resume is not None else None,
                         C.byref(kind))
        if not h:
            msg = L.wref_last_error().decode()
            raise (ValueError if kind.value == 1 else RuntimeError)(msg)
        return Reference(handle=h)

    def deform_backward(self, pos01, up):
        """DeformGrads for upstream dL/d(residuals) up = (d_center, d_response, d_atten)."""
        shapes = self.sc.layer_shapes()
        gw = [np.zeros(s, np.float32) for s in shapes]
        gb = [np.zeros(s[0], np.float32) for s in shapes]
        uc, ur, ua = (_c32(u) for u in up)
        self._check(self.lib.wref_deform_backward(self.h, _f(_c32(pos01)), _f(uc), _f(ur), _f(ua),
                                                  (_fp * 11)(*[_f(w) for w in gw]), (_fp * 11)(*[_f(b) for b in gb])))
        return gw, gb

    def iteration(self):
        self.lib.wref_ck_iteration.restype = C.c_longlong
        return int(self.lib.wref_ck_iteration(self.h))

    def set_iteration(self, it):
        self.lib.wref_ck_set_iteration(self.h, C.c_longlong(it))

    def gradients(self, target, lambda1, pos01=None):
        """The training iteration's gradient chain at these parameters (fine when pos01 given)."""
        sc = self.sc
        n = sc.n
        widths = (2, 3, 1, 2, 2, 2, 1)
        names = ("center_raw", "cholesky", "atten_logit", "response", "d_center", "d_response", "d_atten")
        flat = np.zeros(n * sum(widths), np.float32)
        terms = np.zeros(3)
        shapes = sc.layer_shapes()
        gw = [np.zeros(s, np.float32) for s in shapes]
        gb = [np.zeros(s[0], np.float32) for s in shapes]
        pw = (_fp * 11)(*[_f(w) for w in gw])
        pb = (_fp * 11)(*[_f(b) for b in gb])
        p = None if pos01 is None else _c32(pos01)
        self._check(self.lib.wref_gradients(self.h, _f(p), _f(_c32(target)), C.c_double(lambda1), _d(terms),
                                            _f(flat), pw, pb))
        out, at = {"terms": terms}, 0
        for k, w in zip(names, widths):
            v = flat[at:at + n * w]
            out[k] = v.reshape(n, w) if w > 1 else v.copy()
            at += n * w
        if p is not None:
            out["layer_w"], out["layer_b"] = gw, gb
        return out

    def materialize_center(self, rel, raz, double=False):
        if double:
            el, az = C.c_double(), C.c_double()
            self.lib.wref_materialize_center_d(C.c_double(rel), C.c_double(raz), C.byref(el), C.byref(az))
        else:
            el, az = C.c_float(), C.c_float()
            self.lib.wref_materialize_center_f(C.c_float(rel), C.c_float(raz), C.byref(el), C.byref(az))
        return el.value, az.value


def make_dataset(dataset_dir, H, W, count, seed):
    """Simulate + save a dataset with the reference's own wavesim / dataset code
    (dataset.cpp:61-203); returns (manifest hash, bbox [6])."""
    L = C.CDLL(REF_SO)
    h = C.c_uint64()
    bbox = np.zeros(6)
    if L.wref_make_dataset(dataset_dir.encode(), H, W, count, C.c_uint64(seed), C.byref(h), _d(bbox)) != 0:
        L.wref_last_error.restype = C.c_char_p
        raise RuntimeError(L.wref_last_error().decode())
    return h.value, bbox


def load_dataset(dataset_dir, H, W):
    """The reference's load_dataset (dataset.cpp:205-258): (hash, positions, spectra)."""
    L = C.CDLL(REF_SO)
    L.wref_dataset_load.restype = C.c_longlong
    h = C.c_uint64()
    n = L.wref_dataset_load(dataset_dir.encode(), C.byref(h), None, None, C.c_longlong(0))
    if n < 0:
        L.wref_last_error.restype = C.c_char_p
        raise RuntimeError(L.wref_last_error().decode())
    pos = np.zeros((n, 3), np.float32)
    spec = np.zeros((n, H, W, 2), np.float32)
    L.wref_dataset_load(dataset_dir.encode(), C.byref(h), _f(pos), _f(spec), C.c_longlong(n))
    return h.value, pos, spec


def ref_steering_table(H, W, k=16, spacing=0.0625, wavelength=0.125, nofma=False):
    """build_steering_table through the reference library."""
    L = C.CDLL(REF_NOFMA_SO if nofma else REF_SO)
    wr = np.zeros((H * W, k))
    wi = np.zeros_like(wr)
    if L.wref_steering_table(k, C.c_double(spacing), C.c_double(wavelength), H, W, _d(wr), _d(wi)) != 0:
        raise RuntimeError("wref_steering_table failed")
    return wr, wi


def ref_beam_scan(channel, H, W, k=16, spacing=0.0625, wavelength=0.125, nofma=False):
    """sim::beam_scan(channel, array, grid) -> [H][W][2] float64."""
    L = C.CDLL(REF_NOFMA_SO if nofma else REF_SO)
    ch = np.ascontiguousarray(np.asarray(channel, np.complex128).reshape(k))
    out = np.zeros((H, W, 2))
    if L.wref_beam_scan(k, C.c_double(spacing), C.c_double(wavelength), H, W, _d(ch.view(np.float64)), _d(out)) != 0:
        raise RuntimeError("wref_beam_scan failed")
    return out


def ref_sample_channels(count, seed):
    """The channels generate_dataset scans for make_dataset(dir, H, W, count, seed)."""
    L = C.CDLL(REF_SO)
    ch = np.zeros((count, 16), np.complex128)
    valid = np.zeros(count, np.int32)
    if L.wref_sample_channels(count, C.c_ulonglong(seed), _d(ch.view(np.float64)), _i(valid)) != 0:
        raise RuntimeError("wref_sample_channels failed")
    return ch, valid.astype(bool)
