"""Render backward: splat::rasterize_backward and
train::hybrid_loss on the GPU against the reference compiled from its own
sources (oracle/_ref, built by oracle/Makefile; the shim exposes
wref_rasterize_backward / wref_hybrid_loss).

Contract:
  * gradients: per RenderGrads field, max |GPU - ref| <= 1e-5 * max(1e-6, max |ref|)
    (both FP32; the GPU sums a tile's cells in a different order than the
    reference's row-major loop, splat.cpp:560-640, while the per-tile partials are
    merged in the same ascending tile order, splat.cpp:645-669);
  * entries of primitives that touch no cell stay exactly zero (splat.hpp:74);
  * hybrid loss terms: |GPU - ref| <= 1e-9 (double statistics both sides);
    dLoss/dprediction: max |GPU - ref| <= 1e-6 * max |ref| + 1e-12.
"""
import numpy as np
import pytest

import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions

pytestmark = pytest.mark.gpu
GRAD_TOL = 1e-5


@pytest.fixture(scope="module")
def scene():
    return make_scene(1500, seed=5)


@pytest.fixture(scope="module")
def ck(scene):
    return swr.Checkpoint.from_scene(scene)


@pytest.fixture(scope="module")
def ref(scene):
    return O.Reference(scene)


def _close(got, want, name):
    scale = max(1e-6, float(np.abs(want).max()))
    err = float(np.abs(got - want).max())
    assert err <= GRAD_TOL * scale, f"{name}: max err {err:.3e} vs scale {scale:.3e}"


def _ref_residuals(ref, positions):
    out = [ref.predict(ref.normalize(p)) for p in positions]
    return swr.Residuals(np.stack([o[0] for o in out]), np.stack([o[1] for o in out]), np.stack([o[2] for o in out]))


@pytest.mark.parametrize("with_res", [False, True])
def test_rasterize_backward_matches_reference(scene, ck, ref, with_res):
    rng = np.random.default_rng(3)
    B = 3
    pos = random_positions(B, seed=21)
    res = _ref_residuals(ref, pos) if with_res else None
    up = rng.standard_normal((B, scene.H, scene.W, 2)).astype(np.float32)
    got = swr.rasterize_backward(ck, up, res)
    for b in range(B):
        r = (res.d_center[b], res.d_response[b], res.d_atten[b]) if with_res else None
        want = ref.rasterize_backward(up[b], r)
        for k, _ in swr.GRAD_FIELDS:  # without residuals d_* are the gradients at zero residuals
            _close(got[k][b], want[k], k)
            # primitives that influence no cell: exactly zero on both sides
            zero = np.all(want[k].reshape(scene.n, -1) == 0, axis=1)
            assert np.all(got[k][b].reshape(scene.n, -1)[zero] == 0), k


def test_backward_of_hybrid_loss_matches_reference(scene, ck, ref):
    """The training step's chain: render -> hybrid loss gradient -> rasterize_backward."""
    pos = random_positions(2, seed=8)
    res = _ref_residuals(ref, pos)
    pred = swr.rasterize(ck, res)
    target = np.roll(pred, 7, axis=2) * 0.9
    terms, g = swr.hybrid_loss(ck, pred, target, 0.8)
    for b in range(2):
        wt, wg = ref.hybrid_loss(pred[b], target[b], 0.8)
        assert np.abs(terms[b] - wt).max() <= 1e-9
        assert np.abs(g[b] - wg).max() <= 1e-6 * np.abs(wg).max() + 1e-12
    got = swr.rasterize_backward(ck, g, res)
    for b in range(2):
        want = ref.rasterize_backward(g[b], (res.d_center[b], res.d_response[b], res.d_atten[b]))
        for k, _ in swr.GRAD_FIELDS:
            _close(got[k][b], want[k], k)


@pytest.mark.parametrize("lam", [0.0, 0.8, 1.0])
def test_hybrid_loss_matches_reference(scene, ck, ref, lam):
    rng = np.random.default_rng(11)
    a = rng.standard_normal((3, scene.H, scene.W, 2)).astype(np.float32) * 0.1
    b = a + rng.standard_normal(a.shape).astype(np.float32) * 0.02
    b[2] = a[2]  # identical pair: sign(0) = 0 in the L1 gradient, SSIM = 1
    terms, g = swr.hybrid_loss(ck, a, b, lam)
    t_only, none = swr.hybrid_loss(ck, a, b, lam, grad=False)
    assert none is None and np.array_equal(t_only, terms)
    for i in range(3):
        wt, wg = ref.hybrid_loss(a[i], b[i], lam)
        assert np.abs(terms[i] - wt).max() <= 1e-9, (terms[i], wt)
        assert np.abs(g[i] - wg).max() <= 1e-6 * np.abs(wg).max() + 1e-12


def test_hybrid_loss_errors(scene, ck):
    a = np.zeros((1, scene.H, scene.W, 2), np.float32)
    b = a.copy()
    b[0, 3, 4, 1] = np.nan
    with pytest.raises(ArithmeticError):
        swr.hybrid_loss(ck, a, b, 0.8)
    with pytest.raises(ValueError):
        swr.hybrid_loss(ck, a, b[:, :-1], 0.8)


def test_backward_linear_in_upstream_and_chunking(scene, ck):
    """Gradients are linear in dL/dA (every field is a sum of upstream-weighted
    terms); the chunk size must not change a bit."""
    rng = np.random.default_rng(4)
    up = rng.standard_normal((5, scene.H, scene.W, 2)).astype(np.float32)
    full = swr.rasterize_backward(ck, up)
    zero = swr.rasterize_backward(ck, np.zeros_like(up))
    for k, _ in swr.GRAD_FIELDS:
        assert not np.any(zero[k]), k
    twice = swr.rasterize_backward(ck, up * 2)
    for k, _ in swr.GRAD_FIELDS:
        assert np.array_equal(twice[k], full[k] * 2), k  # power-of-two scaling is exact
    ck2 = swr.Checkpoint.from_scene(scene)
    ck2.set_option("chunk", 2)
    again = swr.rasterize_backward(ck2, up)
    for k, _ in swr.GRAD_FIELDS:
        assert np.array_equal(again[k], full[k]), k
    assert swr.rasterize_backward(ck, up[:0])["center_raw"].shape == (0, scene.n, 2)
