"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref is built):

    python tests/golden/make_golden.py

Every expected value in the fixtures comes out of oracle/_ref/libwrfref*.so,
i.e. the reference's own sources (splat.cpp, training.cpp, tasks.cpp,
checkpoint.cpp, ...) compiled by oracle/Makefile, called through their public
API (load_checkpoint, normalize_position, predict_residuals, rasterize with its
workspace, render_at, aoa_extract, pooled_magnitude). The GPU box has no
/root/reference; tests read these committed files instead.

Fixtures:
  scene_w32.wrfc         90x360 grid, 600 Gaussians, width-32 deform net (WRFC as
                         written by the reference's save_checkpoint)
  golden_w32.npz         positions, residuals, state/rows/cols/bins (contraction-off
                         build), spectra + heads (reference as shipped), canonical render
  criterion1.npz         the acceptance-criterion-1 style small instances (grid <= 16x32,
                         n <= 64, cutoff off, half with residuals) and the reference spectra
  criterion1_ref.npz     the reference's OWN criterion-1 instances: its wrfsplat::Rng(20250814)
                         stream replayed in the shim (acceptance.cpp:130-147, 159-199), with
                         the reference's tiled float rasterize and the criterion's FP64 dense
                         oracle (acceptance.cpp:53-109) for each
  rssi_model_w32.wrfc    scene_w32 saved as an RSSI model by the reference's save_rssi_model
                         (tasks.cpp:131-137): rssi_slope / rssi_intercept in the trailer
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_2506_12787_b200.scene import Scene, make_scene, random_positions, write_wrfc  # noqa: E402


def main():
    O.build(ref=True)
    sc = make_scene(600, seed=2024, width=32)
    tmp = os.path.join(HERE, "_tmp.wrfc")
    write_wrfc(tmp, sc)
    ref = O.Reference(path=tmp)
    ref.save(os.path.join(HERE, "scene_w32.wrfc"))  # written by the reference itself
    os.remove(tmp)
    ref = O.Reference(path=os.path.join(HERE, "scene_w32.wrfc"))
    refn = O.Reference(path=os.path.join(HERE, "scene_w32.wrfc"), nofma=True)
    pos = random_positions(3, seed=5)
    pos01 = np.stack([ref.normalize(p) for p in pos])
    res = [ref.predict(p) for p in pos01]
    d = dict(pos_m=pos, pos01=pos01,
             d_center=np.stack([r[0] for r in res]), d_response=np.stack([r[1] for r in res]),
             d_atten=np.stack([r[2] for r in res]))
    spectra, ws = [], []
    for b in range(3):
        _, w = refn.rasterize(res[b], workspace=True)
        ws.append(w)
        spectra.append(ref.render_at(pos[b]))
    d["spectra"] = np.stack(spectra)
    for k in ("state", "rows", "cols", "tile_offset"):
        d[k] = np.stack([w[k] for w in ws])
    d["tile_prims_len"] = np.array([len(w["tile_prims"]) for w in ws])
    d["tile_prims"] = np.concatenate([w["tile_prims"] for w in ws])
    d["aoa"] = np.array([ref.aoa(s)[:2] for s in spectra], np.int32)
    d["aoa_ang"] = np.array([ref.aoa(s)[2:] for s in spectra], np.float64)
    d["pooled"] = np.array([ref.pooled(s) for s in spectra], np.float64)
    canon, cw = refn.rasterize(None, workspace=True)
    d["canonical"] = ref.rasterize(None)
    d["canonical_tile_offset"] = cw["tile_offset"]
    d["canonical_tile_prims"] = cw["tile_prims"]
    np.savez_compressed(os.path.join(HERE, "golden_w32.npz"), **d)

    # criterion 1 style instances (acceptance.cpp:159-199): cutoff off, small grids
    rng = np.random.default_rng(20250814)
    inst = []
    for i in range(50):
        H, W = 4 + int(rng.integers(13)), 8 + int(rng.integers(25))
        n = 1 + int(rng.integers(64))
        s = Scene(H=H, W=W, center_raw=rng.uniform(-1.5, 1.5, (n, 2)).astype(np.float32),
                  cholesky=np.stack([rng.uniform(0.05, 0.4, n), rng.uniform(-0.2, 0.2, n),
                                     rng.uniform(0.05, 0.4, n)], 1).astype(np.float32),
                  atten_logit=rng.uniform(-1, 1, n).astype(np.float32),
                  response=rng.uniform(-0.5, 0.5, (n, 2)).astype(np.float32), cutoff=0.0)
        r = None
        if i % 2 == 1:
            r = (rng.uniform(-0.05, 0.05, (n, 2)).astype(np.float32), rng.uniform(-0.05, 0.05, (n, 2)).astype(np.float32),
                 rng.uniform(-0.05, 0.05, n).astype(np.float32))
        out = O.Reference(scene=s).rasterize(r)
        inst.append((s, r, out))
    c = {}
    for i, (s, r, out) in enumerate(inst):
        c[f"{i}_hw"] = np.array([s.H, s.W])
        c[f"{i}_cr"], c[f"{i}_ch"], c[f"{i}_at"], c[f"{i}_rs"] = s.center_raw, s.cholesky, s.atten_logit, s.response
        if r is not None:
            c[f"{i}_dc"], c[f"{i}_dr"], c[f"{i}_da"] = r
        c[f"{i}_out"] = out
    np.savez_compressed(os.path.join(HERE, "criterion1.npz"), **c)
    criterion1_ref()
    rssi_model()
    print("golden fixtures written")


def rssi_model():
    ref = O.Reference(path=os.path.join(HERE, "scene_w32.wrfc"))
    out = os.path.join(HERE, "rssi_model_w32.wrfc")
    ref.save_rssi_model(out, 17.25, -58.5)
    assert ref.load_rssi_model(out) == (17.25, -58.5)


def criterion1_ref():
    import ctypes as C
    lib = C.CDLL(O.REF_SO)
    hwn = np.zeros(150, np.int32)
    cr, ch = np.zeros((50, 64, 2), np.float32), np.zeros((50, 64, 3), np.float32)
    at, rs = np.zeros((50, 64), np.float32), np.zeros((50, 64, 2), np.float32)
    dc, dr, da = np.zeros((50, 64, 2), np.float32), np.zeros((50, 64, 2), np.float32), np.zeros((50, 64), np.float32)
    out, dense = np.zeros((50, 1024), np.float32), np.zeros((50, 1024), np.float64)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = lib.wref_criterion1(*[ptr(a) for a in (hwn, cr, ch, at, rs, dc, dr, da, out, dense)])
    assert rc == 0
    np.savez_compressed(os.path.join(HERE, "criterion1_ref.npz"), hwn=hwn.reshape(50, 3), cr=cr, ch=ch, at=at,
                        rs=rs, dc=dc, dr=dr, da=da, out=out, dense=dense)


if __name__ == "__main__":
    if sys.argv[1:]:  # one fixture by name, e.g. `criterion1_ref` or `rssi_model`
        globals()[sys.argv[1]]()
    else:
        main()
