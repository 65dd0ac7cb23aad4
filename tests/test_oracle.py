"""CPU tests: pin the plain-C oracle (oracle/swr_oracle.c) against the reference
itself (oracle/_ref, built from /root/reference sources) and against the golden
vectors in tests/golden/ (also produced by the reference). No GPU needed."""
import math
import os

import numpy as np
import pytest

from conftest import ROOT, has_ref
import oracle as O
from paper_2506_12787_b200.scene import Scene, make_scene, random_positions, read_wrfc, write_wrfc

GOLD = os.path.join(ROOT, "tests", "golden")


def golden_scene():
    return read_wrfc(os.path.join(GOLD, "scene_w32.wrfc"))


def test_materialize_center_kat():
    # test_splat.cpp:146-166
    port = O.Port(golden_scene())
    import ctypes as C
    el, az = C.c_float(), C.c_float()
    port.lib.so_materialize_center(C.c_float(1.0), C.c_float(-1.0), C.byref(el), C.byref(az))
    assert el.value == pytest.approx(1.383552814739336, rel=1e-6)
    assert az.value == pytest.approx(0.7489740482222431, rel=1e-6)
    port.lib.so_materialize_center(C.c_float(0.0), C.c_float(0.0), C.byref(el), C.byref(az))
    assert el.value == pytest.approx(math.pi / 4, rel=1e-7)
    assert az.value == pytest.approx(math.pi, rel=1e-7)


def test_encoding_kat():
    # test_deform.cpp:107-129 (float instantiation)
    port = O.Port(golden_scene())
    vals = np.array([0.25, -0.5], np.float32)
    out = np.full(10, -100, np.float32)
    port.lib.so_encode(O._f(vals), 2, 2, O._f(out))
    want = [0.25, -0.5, math.sin(math.pi / 4), -1.0, math.cos(math.pi / 4), 0.0, 1.0, 0.0, 0.0, -1.0]
    np.testing.assert_allclose(out, want, atol=1e-6)


def test_heads_kats():
    # test_tasks.cpp:67-95
    port = O.Port(golden_scene())
    s = np.zeros((1, 2, 2), np.float32)
    s[0, 0] = [3.0, -4.0]
    assert port.pooled(s) == pytest.approx(2.5, rel=1e-7)
    t = np.zeros((8, 16, 2), np.float32)
    t[2, 9, 1] = 1.5
    t[4, 1, 0] = 1.5
    assert port.aoa(t)[:2] == (2, 9)
    t[2, 5, 0] = 1.5
    assert port.aoa(t)[:2] == (2, 5)


def test_oracle_matches_golden_vectors():
    g = np.load(os.path.join(GOLD, "golden_w32.npz"))
    sc = golden_scene()
    port = O.Port(sc)
    at = 0
    for b in range(3):
        p01 = port.normalize(g["pos_m"][b])
        np.testing.assert_array_equal(p01, g["pos01"][b])
        dc, dr, da = port.predict(p01)
        for got, want in ((dc, g["d_center"][b]), (dr, g["d_response"][b]), (da, g["d_atten"][b])):
            assert np.abs(got - want).max() <= 1e-6 * max(1.0, np.abs(want).max())
        # bins/state from the reference's residuals: bit-exact
        res = (g["d_center"][b], g["d_response"][b], g["d_atten"][b])
        w = port.prepare(res)
        m = int(g["tile_prims_len"][b])
        np.testing.assert_array_equal(w["state"], g["state"][b])
        np.testing.assert_array_equal(w["rows"], g["rows"][b])
        np.testing.assert_array_equal(w["cols"], g["cols"][b])
        np.testing.assert_array_equal(w["tile_offset"], g["tile_offset"][b])
        np.testing.assert_array_equal(w["tile_prims"], g["tile_prims"][at:at + m])
        at += m
        spec = port.rasterize(res, precise=True)
        want = g["spectra"][b]
        assert np.abs(spec - want).max() <= 1e-5 * max(1.0, np.abs(want).max())
        assert port.aoa(want)[:2] == tuple(g["aoa"][b])
        assert port.pooled(want) == pytest.approx(g["pooled"][b], rel=1e-12)
    canon = port.rasterize(None, precise=True)
    assert np.abs(canon - g["canonical"]).max() <= 1e-5


def test_oracle_matches_criterion1_instances():
    c = np.load(os.path.join(GOLD, "criterion1.npz"))
    worst = 0.0
    for i in range(50):
        H, W = map(int, c[f"{i}_hw"])
        s = Scene(H=H, W=W, center_raw=c[f"{i}_cr"], cholesky=c[f"{i}_ch"], atten_logit=c[f"{i}_at"],
                  response=c[f"{i}_rs"], cutoff=0.0)
        r = (c[f"{i}_dc"], c[f"{i}_dr"], c[f"{i}_da"]) if f"{i}_dc" in c else None
        out = O.Port(s).rasterize(r, precise=True)
        worst = max(worst, float(np.abs(out - c[f"{i}_out"]).max()))
    assert worst <= 1e-5


def test_oracle_matches_reference_criterion1_instances():
    """The reference's own criterion-1 instances (Rng(20250814) stream replayed by
    the reference build, tests/golden/make_golden.py criterion1_ref): the port
    meets the gate (<= 1e-5 vs the FP64 dense oracle) and tracks the reference's
    tiled float output."""
    c = np.load(os.path.join(GOLD, "criterion1_ref.npz"))
    worst_dense = worst_ref = 0.0
    for i in range(50):
        H, W, n = map(int, c["hwn"][i])
        s = Scene(H=H, W=W, center_raw=c["cr"][i, :n], cholesky=c["ch"][i, :n], atten_logit=c["at"][i, :n],
                  response=c["rs"][i, :n], cutoff=0.0)
        r = (c["dc"][i, :n], c["dr"][i, :n], c["da"][i, :n]) if i % 2 == 1 else None
        out = O.Port(s).rasterize(r, precise=True).ravel()
        k = 2 * H * W
        worst_dense = max(worst_dense, float(np.abs(out - c["dense"][i, :k]).max()))
        worst_ref = max(worst_ref, float(np.abs(out - c["out"][i, :k]).max()))
    assert worst_dense <= 1e-5 and worst_ref <= 1e-5, (worst_dense, worst_ref)


@pytest.mark.skipif(not has_ref(), reason="reference build absent (GPU box)")
@pytest.mark.parametrize("cutoff,H,W", [(3.0, 90, 360), (0.0, 12, 24), (3.0, 16, 32), (1.5, 45, 90)])
def test_oracle_vs_reference_live(cutoff, H, W):
    sc = make_scene(300, seed=7, H=H, W=W, width=24, cutoff=cutoff)
    ref = O.Reference(scene=sc)
    refn = O.Reference(scene=sc, nofma=True)
    port = O.Port(sc)
    for pos in random_positions(2, seed=3):
        p01 = ref.normalize(pos)
        np.testing.assert_array_equal(p01, port.normalize(pos))
        rres = ref.predict(p01)
        pres = port.predict(p01)
        for a, b in zip(rres, pres):
            assert np.abs(a - b).max() <= 1e-6 * max(1.0, np.abs(a).max())
        _, w = refn.rasterize(rres, workspace=True)
        pw = port.prepare(rres)
        for k in w:
            np.testing.assert_array_equal(w[k], pw[k], err_msg=k)
        # bins are immune to FP contraction
        _, wf = ref.rasterize(rres, workspace=True)
        for k in ("rows", "cols", "tile_offset", "tile_prims"):
            np.testing.assert_array_equal(wf[k], pw[k], err_msg=k)
        spec = ref.render_at(pos)
        mine = port.rasterize(rres, precise=True)
        assert np.abs(spec - mine).max() <= 1e-5 * max(1.0, np.abs(spec).max())


@pytest.mark.skipif(not has_ref(), reason="reference build absent (GPU box)")
def test_wrfc_roundtrip_through_reference(tmp_path):
    sc = make_scene(50, seed=3, width=8, H=16, W=32)
    p = str(tmp_path / "a.wrfc")
    write_wrfc(p, sc)
    ref = O.Reference(path=p)
    p2 = str(tmp_path / "b.wrfc")
    ref.save(p2)
    back = read_wrfc(p2)
    for k in ("center_raw", "cholesky", "atten_logit", "response"):
        np.testing.assert_array_equal(getattr(back, k), getattr(sc, k))
    for a, b in zip(back.weights + back.biases, sc.weights + sc.biases):
        np.testing.assert_array_equal(a, b)
    assert (back.H, back.W, back.cutoff, back.tile) == (sc.H, sc.W, sc.cutoff, sc.tile)
    assert back.bbox_min == pytest.approx(sc.bbox_min) and back.bbox_max == pytest.approx(sc.bbox_max)


def test_dense_fp64_oracle_agrees_with_tiled_oracle():
    # kernel_oracle / dense_oracle of test_splat.cpp:32-106 restated in numpy
    rng = np.random.default_rng(37)
    n, H, W = 20, 12, 24
    s = Scene(H=H, W=W, center_raw=rng.uniform(-1.5, 1.5, (n, 2)).astype(np.float32),
              cholesky=np.stack([rng.uniform(0.05, 0.4, n), rng.uniform(-0.2, 0.2, n), rng.uniform(0.05, 0.4, n)],
                                1).astype(np.float32),
              atten_logit=rng.uniform(-1, 1, n).astype(np.float32),
              response=rng.uniform(-0.5, 0.5, (n, 2)).astype(np.float32), cutoff=0.0)
    want = dense_oracle(s)
    got = O.Port(s).rasterize(None, precise=True)
    assert np.abs(got - want).max() <= 1e-5


def dense_oracle(s, res=None):
    """FP64 dense render (test_splat.cpp:67-106), no cutoff."""
    H, W = s.H, s.W
    el = (np.arange(H) + 0.5) * (math.pi / 2 / H)
    az = (np.arange(W) + 0.5) * (2 * math.pi / W)
    out = np.zeros((H, W, 2))
    for p in range(s.n):
        c_el = math.pi / 4 * (math.tanh(float(s.center_raw[p, 0])) + 1)
        c_az = math.pi * (math.tanh(float(s.center_raw[p, 1])) + 1)
        l1 = max(float(s.cholesky[p, 0]), 1e-4)
        l2 = float(s.cholesky[p, 1])
        l3 = max(float(s.cholesky[p, 2]), 1e-4)
        delta = 1 / (1 + math.exp(-float(s.atten_logit[p])))
        re, im = float(s.response[p, 0]), float(s.response[p, 1])
        if res is not None:
            c_el += float(res[0][p, 0])
            c_az += float(res[0][p, 1])
            re += float(res[1][p, 0])
            im += float(res[1][p, 1])
            delta = min(max(delta + float(res[2][p]), 0.0), 1.0)
        d0 = el[:, None] - c_el
        d1 = np.mod(az[None, :] - c_az + math.pi, 2 * math.pi) - math.pi
        s00, s01, s11 = l1 * l1, l1 * l2, l2 * l2 + l3 * l3
        det = s00 * s11 - s01 * s01
        q = (s11 * d0 * d0 - 2 * s01 * d0 * d1 + s00 * d1 * d1) / det
        k = delta * np.exp(-0.5 * q)
        out[..., 0] += re * k
        out[..., 1] += im * k
    return out


@pytest.mark.skipif(not has_ref(), reason="reference build absent (GPU box)")
def test_reference_backward_shim_field_order():
    """Pins the wref_rasterize_backward wiring: A is linear in response, so
    dL/dresponse_n = sum(upstream * (A(response_n + e) - A)) for L = <upstream, A>,
    and d_response equals response (splat.cpp:494-669)."""
    sc = make_scene(40, seed=2, H=16, W=32, width=24)
    ref = O.Reference(scene=sc)
    rng = np.random.default_rng(0)
    up = rng.standard_normal((16, 32, 2)).astype(np.float32)
    g = ref.rasterize_backward(up)
    assert set(g) == {"center_raw", "cholesky", "atten_logit", "response", "d_center", "d_response", "d_atten"}
    np.testing.assert_array_equal(g["response"], g["d_response"])
    base = ref.rasterize().astype(np.float64)
    for n in (0, 7, 31):
        for c in range(2):
            dr = np.zeros((sc.n, 2), np.float32)
            dr[n, c] = 1.0
            pert = ref.rasterize((np.zeros((sc.n, 2), np.float32), dr, np.zeros(sc.n, np.float32)))
            fd = float(np.sum(up.astype(np.float64) * (pert - base)))
            assert abs(fd - g["response"][n, c]) <= 1e-4 * max(1.0, abs(fd)), (n, c)
    terms, grad = ref.hybrid_loss(base.astype(np.float32), np.zeros((16, 32, 2), np.float32), 0.8)
    assert abs(terms[0] - terms[1] - terms[2]) <= 1e-12 and grad.shape == (16, 32, 2)


@pytest.mark.skipif(not has_ref() or O.blas_library() is None, reason="reference build or numpy OpenBLAS absent")
def test_reference_blas_build_equals_loop_build():
    """The CPU-baseline build of the reference (deform GEMM on a real SGEMM, bench.py
    --impl reference) computes the same residuals and spectra as the restated-loop
    build, bit for bit: both accumulate each output in K order with FMA from zero and
    add the bias afterwards."""
    sc = make_scene(1500, seed=12)
    pos = random_positions(3, seed=13)
    outs = []
    for v in ("loop", "blas"):
        r = O.Reference(scene=sc, variant=v)
        r.set_threads(2)
        outs.append((r.predict(r.normalize(pos[0])), r.render_batch(pos, mode=1, spectra=True)))
    (ra, (sa, pa, ca, _)), (rb, (sb, pb, cb, _)) = outs
    for x, y in zip(ra, rb):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(sa, sb)
    np.testing.assert_array_equal(pa, pb)
    np.testing.assert_array_equal(ca, cb)
