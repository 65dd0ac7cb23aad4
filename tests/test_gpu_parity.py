"""GPU parity: the CUDA path (libswr.so through its C ABI) against the oracle
(oracle/swr_oracle.c, itself pinned to the reference) and the reference's golden
vectors. Contract:

  * render state, row/column ranges, tile counts, CSR tile bins and their
    primitive order: bit-exact (given identical residuals);
  * spectra: max |GPU - oracle| <= 1e-5 * max(1, peak |A|)  (the reference's own
    float-vs-double bar, test_splat.cpp:216-253, acceptance.cpp:159-199);
  * residuals from the FP32 MLP: max |GPU - FP64 oracle| <= 2e-6 * max(1, max|res|);
  * pooled magnitude / RSSI: relative error <= 1e-5; AoA: same cell unless the
    oracle's top two magnitudes are within tolerance.
"""
import os

import numpy as np
import pytest

from conftest import ROOT
import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import Scene, make_scene, random_positions, read_wrfc, write_wrfc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")
SPEC_TOL = 1e-5


def spec_tol(want):
    return SPEC_TOL * max(1.0, float(np.abs(want).max()))


@pytest.fixture(scope="module")
def scene2k():
    sc = make_scene(2000, seed=1)
    sc.rssi_cal = (12.5, -61.0)   # an RSSI model's affine calibration (tasks.cpp:109)
    return sc


@pytest.fixture(scope="module")
def ck2k(scene2k):
    return swr.Checkpoint.from_scene(scene2k)


def residuals_for(port, positions, precise=True):
    out = [port.predict(port.normalize(p), precise=precise) for p in positions]
    return swr.Residuals(np.stack([o[0] for o in out]), np.stack([o[1] for o in out]), np.stack([o[2] for o in out]))


def _res_tuple(res, b):
    return (res.d_center[b], res.d_response[b], res.d_atten[b])


# ---------------------------------------------------------------- setup + bins

@pytest.mark.parametrize("with_res", [False, True])
def test_setup_bit_exact(scene2k, ck2k, with_res):
    port = O.Port(scene2k)
    pos = random_positions(3, seed=11)
    res = residuals_for(port, pos) if with_res else None
    got = swr.setup(ck2k, res, B=3)
    for b in range(3):
        want = port.prepare(_res_tuple(res, b) if with_res else None)
        np.testing.assert_array_equal(got["state"][b], want["state"])
        np.testing.assert_array_equal(got["rows"][b], want["rows"])
        np.testing.assert_array_equal(got["cols"][b], want["cols"])
        counts = np.diff(want["tile_offset"])
        assert got["tile_count"][b].sum() == counts.sum()


def test_bins_bit_exact(scene2k, ck2k):
    port = O.Port(scene2k)
    pos = random_positions(4, seed=12)
    res = residuals_for(port, pos)
    got = swr.bins(ck2k, res)
    for b in range(4):
        want = port.prepare(_res_tuple(res, b))
        np.testing.assert_array_equal(got[b][0], want["tile_offset"])
        np.testing.assert_array_equal(got[b][1], want["tile_prims"])


@pytest.mark.parametrize("cutoff,H,W,tile", [(0.0, 12, 24, 16), (3.0, 16, 32, 8), (1.0, 45, 90, 16),
                                             (3.0, 90, 360, 16), (5.0, 30, 50, 7), (3.0, 90, 360, 32),
                                             (2.0, 40, 100, 24)])
def test_bins_bit_exact_grids(cutoff, H, W, tile):
    sc = make_scene(400, seed=5, H=H, W=W, width=16, cutoff=cutoff, tile=tile)
    ck = swr.Checkpoint.from_scene(sc)
    port = O.Port(sc)
    res = residuals_for(port, random_positions(2, seed=2))
    got = swr.bins(ck, res)
    for b in range(2):
        want = port.prepare(_res_tuple(res, b))
        np.testing.assert_array_equal(got[b][0], want["tile_offset"])
        np.testing.assert_array_equal(got[b][1], want["tile_prims"])
    sp = swr.rasterize(ck, res)
    for b in range(2):
        want = port.rasterize(_res_tuple(res, b), precise=True)
        assert np.abs(sp[b] - want).max() <= spec_tol(want)


def test_edge_primitives_seam_fullcircle_offgrid_dead():
    """Azimuth seam wrap, full-circle boxes, off-grid elevations and delta<=0."""
    n = 64
    rng = np.random.default_rng(3)
    cr = rng.uniform(-2.5, 2.5, (n, 2)).astype(np.float32)
    cr[:16, 1] = rng.choice([-4.0, 4.0, -2.6, 2.6], 16)   # az near 0 / 2pi -> wrapped spans
    ch = np.stack([rng.uniform(0.005, 0.05, n), rng.uniform(-0.02, 0.02, n), rng.uniform(0.005, 0.05, n)],
                  1).astype(np.float32)
    ch[16:20, 2] = 3.0                                      # 2 h_az >= 2 pi: full circle
    ch[20:22, 0] = 1e-7                                     # below the Cholesky floor
    at = rng.uniform(-3, 3, n).astype(np.float32)
    rs = rng.normal(0, 0.1, (n, 2)).astype(np.float32)
    sc = Scene(H=90, W=360, center_raw=cr, cholesky=ch, atten_logit=at, response=rs, width=8)
    from paper_2506_12787_b200.scene import TRUNK
    for i, (r, c) in enumerate(sc.layer_shapes()):
        sc.weights.append(np.zeros((r, c), np.float32))
        sc.biases.append(np.zeros(r, np.float32))
    ck = swr.Checkpoint.from_scene(sc)
    port = O.Port(sc)
    dc = rng.normal(0, 0.05, (2, n, 2)).astype(np.float32)
    dc[0, 30:34, 0] = 2.0                                   # pushed off the elevation range
    dr = rng.normal(0, 0.05, (2, n, 2)).astype(np.float32)
    da = rng.normal(0, 0.3, (2, n)).astype(np.float32)
    da[:, 40:44] = -2.0                                     # delta clamps to 0 -> never binned
    res = swr.Residuals(dc, dr, da)
    st = swr.setup(ck, res)
    got = swr.bins(ck, res)
    sp = swr.rasterize(ck, res)
    for b in range(2):
        want = port.prepare(_res_tuple(res, b))
        np.testing.assert_array_equal(st["state"][b], want["state"])
        np.testing.assert_array_equal(st["rows"][b], want["rows"])
        np.testing.assert_array_equal(st["cols"][b], want["cols"])
        np.testing.assert_array_equal(got[b][0], want["tile_offset"])
        np.testing.assert_array_equal(got[b][1], want["tile_prims"])
        ws = port.rasterize(_res_tuple(res, b), precise=True)
        assert np.abs(sp[b] - ws).max() <= spec_tol(ws)


# ---------------------------------------------------------------------- raster

def test_raster_matches_oracle(scene2k, ck2k):
    port = O.Port(scene2k)
    res = residuals_for(port, random_positions(3, seed=13))
    sp = swr.rasterize(ck2k, res)
    for b in range(3):
        want = port.rasterize(_res_tuple(res, b), precise=True)
        assert np.abs(sp[b] - want).max() <= spec_tol(want)


def test_zero_residuals_bit_identical(scene2k, ck2k):
    n = scene2k.n
    z = swr.Residuals(np.zeros((1, n, 2), np.float32), np.zeros((1, n, 2), np.float32), np.zeros((1, n), np.float32))
    a = swr.rasterize(ck2k, None)
    b = swr.rasterize(ck2k, z)
    assert np.array_equal(a, b)


def test_render_deterministic(scene2k, ck2k):
    pos = random_positions(5, seed=14)
    a = swr.render(ck2k, pos)
    b = swr.render(ck2k, pos)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_criterion1_instances_vs_reference():
    c = np.load(os.path.join(GOLD, "criterion1.npz"))
    worst = 0.0
    for i in range(50):
        H, W = map(int, c[f"{i}_hw"])
        s = Scene(H=H, W=W, center_raw=c[f"{i}_cr"], cholesky=c[f"{i}_ch"], atten_logit=c[f"{i}_at"],
                  response=c[f"{i}_rs"], cutoff=0.0)
        ck = swr.Checkpoint.from_scene(s)
        r = None
        if f"{i}_dc" in c:
            r = swr.Residuals(c[f"{i}_dc"][None], c[f"{i}_dr"][None], c[f"{i}_da"][None])
        out = swr.rasterize(ck, r)[0]
        worst = max(worst, float(np.abs(out - c[f"{i}_out"]).max()))
    assert worst <= 1e-5


def _criterion1_ref_scenes():
    c = np.load(os.path.join(GOLD, "criterion1_ref.npz"))
    for i in range(50):
        H, W, n = map(int, c["hwn"][i])
        s = Scene(H=H, W=W, center_raw=c["cr"][i, :n], cholesky=c["ch"][i, :n], atten_logit=c["at"][i, :n],
                  response=c["rs"][i, :n], cutoff=0.0)
        r = (c["dc"][i, :n], c["dr"][i, :n], c["da"][i, :n]) if i % 2 == 1 else None
        k = 2 * H * W
        yield s, r, c["out"][i, :k].reshape(H, W, 2), c["dense"][i, :k].reshape(H, W, 2)


def test_reference_criterion1_instances():
    """The acceptance gate's own 50 instances (wrfsplat::Rng(20250814),
    acceptance.cpp:159-199, replayed by the reference build): GPU vs the
    criterion's FP64 dense oracle, max |diff| <= 1e-5, and vs the reference's own
    tiled float rasterize."""
    worst_dense = worst_ref = 0.0
    for s, r, out_ref, dense in _criterion1_ref_scenes():
        ck = swr.Checkpoint.from_scene(s)
        res = swr.Residuals(r[0][None], r[1][None], r[2][None]) if r is not None else None
        got = swr.rasterize(ck, res)[0]
        worst_dense = max(worst_dense, float(np.abs(got - dense).max()))
        worst_ref = max(worst_ref, float(np.abs(got - out_ref).max()))
    assert worst_dense <= 1e-5, worst_dense
    assert worst_ref <= 1e-5, worst_ref


# ------------------------------------------------------------------------- MLP

def test_mlp_fp32_matches_fp64_oracle(scene2k, ck2k):
    port = O.Port(scene2k)
    pos = random_positions(3, seed=15)
    p01 = np.stack([port.normalize(p) for p in pos])
    got = swr.predict_residuals(ck2k, p01)
    for b in range(3):
        want = port.predict(p01[b], precise=True)
        for g, w in zip((got.d_center[b], got.d_response[b], got.d_atten[b]), want):
            assert np.abs(g - w).max() <= 2e-6 * max(1.0, float(np.abs(w).max()))


def test_normalize_matches_reference_bits(scene2k, ck2k):
    port = O.Port(scene2k)
    pos = random_positions(16, seed=16)
    got = swr.normalize_position(ck2k, pos)
    want = np.stack([port.normalize(p) for p in pos])
    np.testing.assert_array_equal(got, want)


# ------------------------------------------------------------------ end to end

def test_render_end_to_end(scene2k, ck2k):
    """FP32 MLP end to end against the oracle (FP64 MLP + FP64 raster). Cells whose
    cutoff mask or bin flips between the two residual sets may differ by up to
    exp(-4.5) * max |k| (the reference's own FP32 path shows the same effect)."""
    port = O.Port(scene2k)
    pos = random_positions(4, seed=17)
    out = swr.render(ck2k, pos, rssi=True)
    kmax = float(np.abs(scene2k.response).max()) + 0.2
    for b in range(4):
        want, _ = port.render(pos[b], precise=True)
        err = np.abs(out["spectra"][b] - want)
        assert np.quantile(err, 0.999) <= spec_tol(want)
        assert err.max() <= np.exp(-4.5) * kmax + spec_tol(want)
        assert out["pooled"][b] == pytest.approx(port.pooled(want), rel=1e-5)
        r, c, el, az = port.aoa(want)
        if tuple(out["aoa_rc"][b]) != (r, c):
            mag = np.hypot(want[..., 0].astype(np.float64), want[..., 1])
            top = np.sort(mag.ravel())[-2:]
            assert top[1] - top[0] <= spec_tol(want)
        else:
            assert out["aoa_ang"][b] == pytest.approx([el, az], abs=1e-12)
    # GPU heads on the GPU spectra agree exactly with the oracle's heads on them
    pooled, rc, ang = swr.heads(ck2k, out["spectra"])
    for b in range(4):
        assert tuple(rc[b]) == port.aoa(out["spectra"][b])[:2]
        assert pooled[b] == pytest.approx(port.pooled(out["spectra"][b]), rel=1e-12)
        assert tuple(out["aoa_rc"][b]) == tuple(rc[b])


def test_golden_vectors_from_reference(tmp_path):
    g = np.load(os.path.join(GOLD, "golden_w32.npz"))
    ck = swr.load_checkpoint(os.path.join(GOLD, "scene_w32.wrfc"))
    p01 = swr.normalize_position(ck, g["pos_m"])
    np.testing.assert_array_equal(p01, g["pos01"])
    res = swr.predict_residuals(ck, p01)
    for got, want in ((res.d_center, g["d_center"]), (res.d_response, g["d_response"]), (res.d_atten, g["d_atten"])):
        assert np.abs(got - want).max() <= 2e-6 * max(1.0, np.abs(want).max())
    # state / bins from the reference's own residuals: bit-exact
    gres = swr.Residuals(g["d_center"], g["d_response"], g["d_atten"])
    st = swr.setup(ck, gres)
    np.testing.assert_array_equal(st["state"], g["state"])
    np.testing.assert_array_equal(st["rows"], g["rows"])
    np.testing.assert_array_equal(st["cols"], g["cols"])
    bins = swr.bins(ck, gres)
    at = 0
    for b in range(3):
        m = int(g["tile_prims_len"][b])
        np.testing.assert_array_equal(bins[b][0], g["tile_offset"][b])
        np.testing.assert_array_equal(bins[b][1], g["tile_prims"][at:at + m])
        at += m
    out = swr.render(ck, g["pos_m"])
    for b in range(3):
        assert np.abs(out["spectra"][b] - g["spectra"][b]).max() <= spec_tol(g["spectra"][b])
        assert tuple(out["aoa_rc"][b]) == tuple(g["aoa"][b])
        assert out["pooled"][b] == pytest.approx(g["pooled"][b], rel=1e-5)
    canon = swr.render(ck, g["pos_m"][:1], residuals=False)["spectra"][0]
    assert np.abs(canon - g["canonical"]).max() <= spec_tol(g["canonical"])
    cb = swr.bins(ck, None)
    np.testing.assert_array_equal(cb[0][0], g["canonical_tile_offset"])
    np.testing.assert_array_equal(cb[0][1], g["canonical_tile_prims"])


def test_rssi_model_from_reference_trailer():
    """An RSSI model saved by the reference (save_rssi_model): the calibration comes
    from its trailer (load_rssi_model, tasks.cpp:139-150) and RSSI is
    slope * pooled + intercept (eval_rssi, tasks.cpp:109), pooled matching the
    reference's pooled_magnitude of its own render_at within 1e-5."""
    ck = swr.load_checkpoint(os.path.join(GOLD, "rssi_model_w32.wrfc"))
    assert ck.get_option("rssi_calibrated") == 1
    assert (ck.get_option("rssi_slope"), ck.get_option("rssi_intercept")) == (17.25, -58.5)
    g = np.load(os.path.join(GOLD, "golden_w32.npz"))
    out = swr.render(ck, g["pos_m"], rssi=True)
    np.testing.assert_allclose(out["rssi"], 17.25 * out["pooled"] - 58.5, rtol=1e-15, atol=0)
    np.testing.assert_allclose(out["pooled"], g["pooled"], rtol=1e-5)
    np.testing.assert_allclose(out["rssi"], 17.25 * g["pooled"] - 58.5, rtol=1e-5)


def test_rssi_requires_a_calibration():
    """A plain checkpoint is not an RSSI model: asking for RSSI fails the way
    load_rssi_model does (runtime_error), until the calibration is set."""
    ck = swr.load_checkpoint(os.path.join(GOLD, "scene_w32.wrfc"))
    assert ck.get_option("rssi_calibrated") == 0
    pos = random_positions(2, seed=1)
    with pytest.raises(swr.SwrError):
        swr.render(ck, pos, rssi=True)
    swr.render(ck, pos)            # everything else renders
    ck.set_option("rssi_slope", 2.0)
    ck.set_option("rssi_intercept", 1.0)
    out = swr.render(ck, pos, rssi=True)
    np.testing.assert_allclose(out["rssi"], 2.0 * out["pooled"] + 1.0, rtol=1e-15)


def test_chunking_invariance(scene2k):
    ck = swr.Checkpoint.from_scene(scene2k)
    pos = random_positions(37, seed=18)
    a = swr.render(ck, pos)
    ck.set_option("chunk", 5)
    b = swr.render(ck, pos)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_device_api_matches_host_api(scene2k, ck2k):
    torch = pytest.importorskip("torch")
    pos = random_positions(6, seed=19)
    host = swr.render(ck2k, pos, rssi=True)
    d_pos = torch.from_numpy(pos).cuda()
    d_spec = torch.zeros((6, ck2k.H, ck2k.W, 2), dtype=torch.float32, device="cuda")
    d_pooled = torch.zeros(6, dtype=torch.float64, device="cuda")
    d_rc = torch.zeros((6, 2), dtype=torch.int32, device="cuda")
    flags = swr.OUT_SPECTRA | swr.OUT_POOLED | swr.OUT_AOA
    stream = torch.cuda.current_stream().cuda_stream
    swr.render_device(ck2k, d_pos.data_ptr(), 6, flags, d_spec.data_ptr(), d_pooled.data_ptr(), 0, d_rc.data_ptr(),
                      0, stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_spec.cpu().numpy(), host["spectra"])
    assert np.array_equal(d_pooled.cpu().numpy(), host["pooled"])
    assert np.array_equal(d_rc.cpu().numpy(), host["aoa_rc"])


def test_errors_follow_reference_types(tmp_path, scene2k):
    sc = make_scene(10, seed=1, width=8, H=16, W=32)
    p = str(tmp_path / "s.wrfc")
    write_wrfc(p, sc)
    ck = swr.load_checkpoint(p)
    with pytest.raises(ValueError):
        ck.set_option("no_such_option", 1)
    bad = tmp_path / "bad.wrfc"
    bad.write_bytes(open(p, "rb").read()[:40])
    with pytest.raises(swr.SwrError):
        swr.load_checkpoint(str(bad))
    with pytest.raises(ValueError):
        swr.Checkpoint.from_scene(Scene(H=0, W=10, center_raw=sc.center_raw, cholesky=sc.cholesky,
                                        atten_logit=sc.atten_logit, response=sc.response))


def test_empty_gaussian_set_follows_the_reference():
    """n = 0: render_at's predict_residuals throws invalid_argument("empty gaussian
    set") (deform.cpp:147-148); rasterize without residuals gives the all-zero
    spectrum (and its heads: pooled 0, AoA at the first cell, RSSI = intercept)."""
    import dataclasses
    base = make_scene(10, seed=1, width=16)
    base.rssi_cal = (2.0, -50.0)
    empty = dataclasses.replace(base, center_raw=base.center_raw[:0], cholesky=base.cholesky[:0],
                                atten_logit=base.atten_logit[:0], response=base.response[:0])
    pos = random_positions(3, seed=2)
    ck = swr.Checkpoint.from_scene(empty)
    with pytest.raises(ValueError, match="empty gaussian set"):
        swr.render(ck, pos, rssi=True)
    for sc, kw in ((empty, dict(residuals=False)), (dataclasses.replace(empty, weights=[], biases=[]), {})):
        out = swr.render(swr.Checkpoint.from_scene(sc), pos, rssi=True, **kw)
        assert out["spectra"].shape == (3, sc.H, sc.W, 2) and not out["spectra"].any()
        assert not out["pooled"].any()
        assert np.all(out["rssi"] == -50.0)
        port = O.Port(sc)
        assert not port.rasterize().any()
        r, c, el, az = port.aoa(np.zeros((sc.H, sc.W, 2), np.float32))
        assert np.all(out["aoa_rc"] == (r, c))
        assert np.all(out["aoa_ang"] == (el, az))


def test_nonfinite_positions_are_contained(scene2k, ck2k):
    """NaN / inf / 1e30 TX positions (undefined behaviour in the reference) neither
    trap nor hang (the checked build runs this too) and leave the finite positions
    of the batch at their own render's value: identical bits when their chunk holds
    no bad position, within the FP32-grade bar where the bad neighbour made the
    chunk re-run its MLP in FP32."""
    pos = random_positions(40, seed=3)
    bad = [1, 2, 3, 4, 5]
    pos[1] = np.nan
    pos[2, 0] = np.inf
    pos[3] = -np.inf
    pos[4] = 1e30
    pos[5] = -1e30
    ck = swr.Checkpoint.from_scene(scene2k)
    ck.set_option("chunk", 16)
    out = swr.render(ck, pos)
    assert out["spectra"].shape == (40, scene2k.H, scene2k.W, 2)
    good = [i for i in range(40) if i not in bad]
    alone = swr.render(ck, pos[good])
    for j, i in enumerate(good):
        a, b = out["spectra"][i], alone["spectra"][j]
        if i >= 16:                                  # chunks without a bad position: same kernels, same bits
            assert np.array_equal(a, b), i
        else:
            assert np.abs(a - b).max() <= spec_tol(b), i


# ---------------------------------------------------------- tensor-core MLP

def _mlp_errors(ck, port, p01, idx):
    """(worst absolute error / max(1, field max), worst error / field max) of the
    residuals against the FP64 oracle over positions idx."""
    got = swr.predict_residuals(ck, p01)
    worst_abs = worst_rel = 0.0
    for b in idx:
        want = port.predict(p01[b], precise=True)
        for g, w in zip((got.d_center[b], got.d_response[b], got.d_atten[b]), want):
            e = float(np.abs(g - w).max())
            m = float(np.abs(w).max())
            worst_abs = max(worst_abs, e / max(1.0, m))
            worst_rel = max(worst_rel, e / max(1e-30, m))
    return worst_abs, worst_rel


def test_mlp_tensor_core_fp32_grade(scene2k):
    """FP16X3 (the tensor-core default): the FP32 bar of test_mlp_fp32_matches_fp64_oracle
    (2e-6 * max(1, |res|)) and, relative to each field's largest residual, within 4x of
    the FP32 CUDA-core kernel's own error against FP64 (deform.cpp:126-137 is FP32)."""
    port = O.Port(scene2k)
    pos = random_positions(13, seed=21)          # odd tile count: exercises the masked tail pair
    p01 = np.stack([port.normalize(p) for p in pos])
    ck32 = swr.Checkpoint.from_scene(scene2k)
    ck32.set_option("mlp_precision", swr.MLP_FP32)
    ck16 = swr.Checkpoint.from_scene(scene2k)
    ck16.set_option("mlp_precision", swr.MLP_FP16X3)
    a32, r32 = _mlp_errors(ck32, port, p01, range(13))
    a16, r16 = _mlp_errors(ck16, port, p01, range(13))
    print(f"fp32 simt: abs {a32:.3g} rel {r32:.3g}; fp16x3: abs {a16:.3g} rel {r16:.3g}")
    assert a16 <= 2e-6, a16
    assert r16 <= max(4.0 * r32, 1e-6), (r16, r32)
    assert ck16.get_option("mlp_reruns") == 0


def test_mlp_tensor_core_single_pass_tier(scene2k):
    ck = swr.Checkpoint.from_scene(scene2k)
    ck.set_option("mlp_precision", swr.MLP_FP16)
    port = O.Port(scene2k)
    pos = random_positions(5, seed=21)
    p01 = np.stack([port.normalize(p) for p in pos])
    _, rel = _mlp_errors(ck, port, p01, range(5))
    assert rel <= 5e-3, rel


def test_mlp_tensor_core_many_tiles(scene2k):
    """Many tiles per CTA pair (203 positions x 2k Gaussians: ~11 super-tiles per pair,
    a ragged last position block), against the FP64 oracle at the FP32 bar."""
    ck = swr.Checkpoint.from_scene(scene2k)
    ck.set_option("mlp_precision", swr.MLP_FP16X3)
    port = O.Port(scene2k)
    pos = random_positions(203, seed=23)
    p01 = np.stack([port.normalize(p) for p in pos])
    a16, _ = _mlp_errors(ck, port, p01, range(0, 203, 7))
    assert a16 <= 2e-6, a16


def test_mlp_activation_scale_adapts_to_the_net():
    """Large activations (layer-1 outputs ~1e5, beyond fp16's 65504): the scene-load
    probe picks a negative activation scale, so the tensor-core path stays on the
    tensor cores and within the FP32 bar of the FP64 oracle."""
    sc = make_scene(300, seed=9)
    sc.weights[1] = (sc.weights[1] * 3e5).astype(np.float32)
    sc.weights[3] = (sc.weights[3] * 3e-6).astype(np.float32)   # back to O(1) after layer 3
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("mlp_precision", swr.MLP_FP16X3)
    assert ck.get_option("mlp_probe_amax") > 65504.0 / 64
    assert ck.get_option("mlp_act_scale_exp") < 0
    port = O.Port(sc)
    p01 = np.stack([port.normalize(p) for p in random_positions(4, seed=3)])
    a16, _ = _mlp_errors(ck, port, p01, range(4))
    assert a16 <= 2e-6, a16
    assert ck.get_option("mlp_reruns") == 0


def test_mlp_fp16_overflow_reruns_in_fp32(scene2k):
    """Positions far outside the training bbox (the encoding's raw coordinates ~1e4,
    activations the scene-load probe never saw) overflow fp16; the NaN reaches the
    residuals (max.NaN ReLU), the setup kernel flags it and the chunk re-runs on the
    FP32 CUDA-core kernel, so every output equals the FP32 path's bit for bit."""
    ck32 = swr.Checkpoint.from_scene(scene2k)
    ck32.set_option("mlp_precision", swr.MLP_FP32)
    ck16 = swr.Checkpoint.from_scene(scene2k)
    ck16.set_option("mlp_precision", swr.MLP_FP16X3)
    pos = random_positions(20, seed=3)
    pos[5:9] += np.float32(3e4)                      # pos01 ~ 1e4
    a = swr.render(ck32, pos, rssi=True)
    b = swr.render(ck16, pos, rssi=True)
    assert ck16.get_option("mlp_reruns") >= 1
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    p01 = swr.normalize_position(ck16, pos[4:10])
    r32 = swr.predict_residuals(ck32, p01)
    n0 = ck16.get_option("mlp_reruns")
    r16 = swr.predict_residuals(ck16, p01)
    assert ck16.get_option("mlp_reruns") > n0
    assert np.array_equal(r32.d_center, r16.d_center) and np.array_equal(r32.d_atten, r16.d_atten)


def test_tensor_core_render_end_to_end(scene2k):
    """FP16X3 MLP end to end. Spectra rendered from the GPU's own residuals match the
    oracle to 1e-5; against the oracle's FP64-MLP render, 99.9% of cells agree to 1e-5
    and the rest are cutoff-mask / bin flips bounded by exp(-4.5) * max |k|; pooled
    within 1e-5 and the AoA cell the same unless the oracle's top two tie."""
    ck = swr.Checkpoint.from_scene(scene2k)
    ck.set_option("mlp_precision", swr.MLP_FP16X3)
    port = O.Port(scene2k)
    pos = random_positions(6, seed=22)
    out = swr.render(ck, pos)
    p01 = np.stack([port.normalize(p) for p in pos])
    res = swr.predict_residuals(ck, p01)
    kmax = float(np.abs(scene2k.response).max()) + 0.2
    for b in range(6):
        own = port.rasterize(_res_tuple(res, b), precise=True)
        assert np.abs(out["spectra"][b] - own).max() <= spec_tol(own)
        want, _ = port.render(pos[b], precise=True)
        err = np.abs(out["spectra"][b] - want)
        assert np.quantile(err, 0.999) <= spec_tol(want)
        assert err.max() <= np.exp(-4.5) * kmax + spec_tol(want)
        assert out["pooled"][b] == pytest.approx(port.pooled(want), rel=1e-5)
        _assert_aoa(out["aoa_rc"][b], want, port)


def _assert_aoa(rc, want, port):
    r, c, _, _ = port.aoa(want)
    if tuple(rc) != (r, c):
        mag = np.hypot(want[..., 0].astype(np.float64), want[..., 1])
        top = np.sort(mag.ravel())[-2:]
        assert top[1] - top[0] <= spec_tol(want), (tuple(rc), (r, c))


def test_render_device_async_overflow_gated_rerun(scene2k):
    """swr_render_device never waits for the host: an fp16 overflow is re-run in FP32
    through kernels gated on the device flag, so the outputs still equal the FP32
    path's bit for bit, and the pair count stays on the device until asked for."""
    import torch
    ck32 = swr.Checkpoint.from_scene(scene2k)
    ck32.set_option("mlp_precision", swr.MLP_FP32)
    ck16 = swr.Checkpoint.from_scene(scene2k)
    ck16.set_option("mlp_precision", swr.MLP_FP16X3)
    ck16.set_option("chunk", 8)
    ckh = swr.Checkpoint.from_scene(scene2k)
    ckh.set_option("mlp_precision", swr.MLP_FP16X3)
    ckh.set_option("chunk", 8)
    pos = random_positions(24, seed=5)
    pos[9:11] += np.float32(3e4)
    want = swr.render(ckh, pos)           # same chunks through the host-buffer entry
    w32 = swr.render(ck32, pos[8:16])     # the overflowing chunk re-runs on the FP32 kernel
    d_pos = torch.from_numpy(pos).cuda()
    d_spec = torch.zeros((24, scene2k.H, scene2k.W, 2), device="cuda")
    d_pooled = torch.zeros(24, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    swr.render_device(ck16, d_pos.data_ptr(), 24, swr.OUT_SPECTRA | swr.OUT_POOLED, d_spec.data_ptr(),
                      d_pooled.data_ptr(), stream=st.cuda_stream)
    st.synchronize()
    assert np.array_equal(d_spec.cpu().numpy(), want["spectra"])
    assert np.array_equal(d_pooled.cpu().numpy(), want["pooled"])
    assert np.array_equal(d_spec.cpu().numpy()[8:16], w32["spectra"])
    assert ck16.get_option("mlp_reruns") == 1          # only the chunk holding the far positions
    assert ck16.pairs_last() > 0


@pytest.mark.parametrize("precision", [swr.MLP_FP16X3, swr.MLP_FP32], ids=["fp16x3", "fp32"])
def test_sync_and_async_chunk_paths_agree(scene2k, precision):
    """Scenes whose pair bound exceeds the per-chunk budget read the pair count back
    and size the bin buffers to it (the round-1 path); the default sizes them to the
    bound and never waits for the host. Both give the same bits, including an
    overflow chunk's FP32 re-run."""
    pos = random_positions(40, seed=14)
    pos[20] += np.float32(3e4)
    outs = []
    for budget in (-1, 0):
        ck = swr.Checkpoint.from_scene(scene2k)
        ck.set_option("mlp_precision", precision)
        ck.set_option("chunk", 16)
        ck.set_option("async_pair_budget", budget)
        outs.append(swr.render(ck, pos, rssi=False))
        assert ck.pairs_last() > 0
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_render_device_cuda_graph_replay(scene2k):
    """swr_render_device captured into a CUDA graph (after one uncaptured call sized
    the buffers): each replay re-reads the position buffer and matches an uncaptured
    call bit for bit -- spectra, pooled, AoA -- including a chunk whose fp16 MLP
    overflows (the device-gated FP32 re-run is part of the graph)."""
    import torch
    flags = swr.OUT_SPECTRA | swr.OUT_POOLED | swr.OUT_AOA
    ck = swr.Checkpoint.from_scene(scene2k)
    ck.set_option("chunk", 8)
    ref = swr.Checkpoint.from_scene(scene2k)
    ref.set_option("chunk", 8)
    B, H, W = 20, scene2k.H, scene2k.W
    st = torch.cuda.Stream()
    d_pos = torch.from_numpy(random_positions(B, seed=40)).cuda()
    outs = dict(spec=torch.zeros((B, H, W, 2), device="cuda"), pooled=torch.zeros(B, dtype=torch.float64, device="cuda"),
                rc=torch.zeros((B, 2), dtype=torch.int32, device="cuda"),
                ang=torch.zeros((B, 2), dtype=torch.float64, device="cuda"))

    def call(c, o):
        swr.render_device(c, d_pos.data_ptr(), B, flags, o["spec"].data_ptr(), o["pooled"].data_ptr(), 0,
                          o["rc"].data_ptr(), o["ang"].data_ptr(), stream=st.cuda_stream)

    with torch.cuda.stream(st):
        call(ck, outs)                      # sizes the work buffers
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            call(ck, outs)
    for seed, far in ((41, False), (42, True), (43, False)):
        p = random_positions(B, seed=seed)
        if far:
            p[9:11] += np.float32(3e4)      # an fp16 overflow in the second chunk
        with torch.cuda.stream(st):
            d_pos.copy_(torch.from_numpy(p))
            for v in outs.values():
                v.zero_()
            g.replay()
            want = {k: torch.zeros_like(v) for k, v in outs.items()}
            call(ref, want)
        st.synchronize()
        for k in outs:
            assert torch.equal(outs[k], want[k]), (seed, k)
        assert float(outs["spec"].abs().max()) > 0
    assert ck.get_option("mlp_reruns") == 1
