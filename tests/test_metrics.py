"""Evaluation metrics: psnr / ssim / l1 of rendered
spectra against targets (spectrum.cpp:145-250) and the batched train::evaluate
(training.cpp:380-406).

CPU: the C restatement (oracle/swr_oracle.c so_metrics) against the reference's
own functions built from its sources (oracle/_ref) and the KATs of
tests/test_spectrum.cpp:110-160. GPU: k_metrics.cu through the C ABI against the
oracle (psnr / l1 relative <= 1e-12, ssim absolute <= 1e-12: all statistics are
double on both sides, only the summation order differs)."""
import numpy as np
import pytest

import oracle as O
from paper_2506_12787_b200.scene import make_scene, random_positions


def _pair(H, W, seed, noise=0.05):
    rng = np.random.default_rng(seed)
    a = (rng.normal(size=(H, W, 2)) * 0.2).astype(np.float32)
    b = (a + rng.normal(size=a.shape) * noise).astype(np.float32)
    return a, b


@pytest.fixture(scope="module")
def port():
    return O.Port(make_scene(50, seed=2))


def test_oracle_kats(port):
    # test_spectrum.cpp:110-143
    a = np.array([[[1.0, 0.0], [0.0, 0.0]]], np.float32)
    b = np.array([[[0.5, 0.0], [0.0, 0.0]]], np.float32)
    p, _, _ = port.metrics(a, b, ssim=False)
    assert abs(p - 12.041199826559248) <= 1e-12 * 12.04
    assert port.metrics(b, a, ssim=False)[0] == p
    x, _ = _pair(12, 16, 7)
    assert port.metrics(x, x, ssim=False)[0] == 100.0
    c = np.array([[[0.25, -0.5]]], np.float32)
    z = np.zeros_like(c)
    assert abs(port.metrics(c, z, ssim=False)[2] - 0.375) <= 1e-15
    assert port.metrics(c, c, ssim=False)[2] == 0.0
    y, _ = _pair(16, 20, 11)
    assert abs(port.metrics(y, y)[1] - 1.0) <= 1e-12


def test_oracle_errors(port):
    a, b = _pair(12, 12, 3)
    a[1, 1, 1] = np.nan
    with pytest.raises(ArithmeticError):
        port.metrics(a, b)
    s, t = _pair(8, 10, 4)
    with pytest.raises(ValueError):
        port.metrics(s, t)
    port.metrics(s, t, ssim=False)  # psnr / l1 have no minimum grid


@pytest.mark.parametrize("H,W,peak", [(16, 24, 1.0), (90, 360, 1.0), (90, 360, 0.5), (23, 41, 3.0)])
def test_oracle_matches_reference(port, H, W, peak):
    ref = O.Reference(make_scene(50, seed=2, H=H, W=W))
    for seed in range(3):
        a, b = _pair(H, W, seed, noise=0.01 * (seed + 1))
        got, want = port.metrics(a, b, peak), ref.metrics(a, b, peak)
        assert abs(got[0] - want[0]) <= 1e-12 * abs(want[0])
        assert abs(got[1] - want[1]) <= 1e-12
        assert abs(got[2] - want[2]) <= 1e-12 * abs(want[2])


@pytest.mark.gpu
def test_gpu_metrics_vs_oracle(port):
    from paper_2506_12787_b200 import swr
    sc = make_scene(64, seed=5)
    ck = swr.Checkpoint.from_scene(sc)
    B = 5
    pairs = [_pair(sc.H, sc.W, 100 + i, noise=0.003 * (i + 1)) for i in range(B)]
    pred = np.stack([p[0] for p in pairs])
    tgt = np.stack([p[1] for p in pairs])
    pred[2] = tgt[2]  # identical pair
    for chunk in (256, 2):
        ck.set_option("chunk", chunk)
        for peak in (1.0, 2.5):
            got = swr.metrics(ck, pred, tgt, peak)
            for i in range(B):
                want = port.metrics(pred[i], tgt[i], peak)
                assert abs(got["psnr"][i] - want[0]) <= 1e-12 * abs(want[0]), (chunk, peak, i)
                assert abs(got["ssim"][i] - want[1]) <= 1e-12, (chunk, peak, i)
                assert abs(got["l1"][i] - want[2]) <= 1e-12 * max(abs(want[2]), 1e-300), (chunk, peak, i)
    assert got["psnr"][2] == 100.0 and got["l1"][2] == 0.0 and abs(got["ssim"][2] - 1.0) <= 1e-12
    # deterministic
    again = swr.metrics(ck, pred, tgt, 2.5)
    for k in got:
        assert np.array_equal(got[k], again[k])


@pytest.mark.gpu
def test_gpu_metrics_errors():
    from paper_2506_12787_b200 import swr
    ck = swr.Checkpoint.from_scene(make_scene(32, seed=5))
    a, b = _pair(ck.H, ck.W, 1)
    a[10, 20, 0] = np.inf
    with pytest.raises(ArithmeticError):
        swr.metrics(ck, a[None], b[None])
    small = swr.Checkpoint.from_scene(make_scene(32, seed=5, H=8, W=10))
    s, t = _pair(8, 10, 2)
    with pytest.raises(ValueError):
        swr.metrics(small, s[None], t[None])
    out = swr.metrics(small, s[None], t[None], ssim=False)
    want = O.Port(make_scene(32, seed=5, H=8, W=10)).metrics(s, t, ssim=False)
    assert abs(out["psnr"][0] - want[0]) <= 1e-12 * abs(want[0])


@pytest.mark.gpu
def test_gpu_evaluate_matches_render_then_metrics():
    from paper_2506_12787_b200 import swr
    sc = make_scene(400, seed=9)
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("mlp_precision", swr.MLP_FP16X3)
    pos = random_positions(7, seed=4)
    spec = swr.render(ck, pos)["spectra"]
    rng = np.random.default_rng(0)
    tgt = (spec + rng.normal(size=spec.shape) * 1e-3).astype(np.float32)
    ck.set_option("chunk", 3)
    ev = swr.evaluate(ck, pos, tgt)
    ref = swr.metrics(ck, spec, tgt)
    for k in ("psnr", "ssim", "l1"):
        assert np.array_equal(ev[k], ref[k]), k
    same = swr.evaluate(ck, pos, spec)
    assert np.all(same["psnr"] == 100.0) and np.all(same["l1"] == 0.0)
    assert np.all(np.abs(same["ssim"] - 1.0) <= 1e-12)
