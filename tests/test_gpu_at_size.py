"""GPU parity at the BASELINE sizes: the reference grid (90 x 360), N = 10k (the
SPEC-sized set, training.hpp:98) and N = 50k (BASELINE config 2), B = 300
positions, so the default position chunks (256 at 50k; forced to 128 at 10k)
and the 2048-pair sort chunks inside every position segment are crossed.

Contract: render state / row / column ranges and the CSR tile
bins with their primitive order bit-exact against the oracle's prepare()
(oracle/swr_oracle.c, pinned to the reference in tests/test_oracle.py) given
identical residuals; spectra within 1e-5 * max(1, peak |A|) of the oracle's
rasterize(); the tensor-core MLP within the FP32 bar of the FP64 oracle; the
batched render equal to rasterize() of its own residuals (chunk plumbing).
"""
import numpy as np
import pytest

import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions

pytestmark = pytest.mark.gpu
B = 300
SPEC_TOL = 1e-5


def spec_tol(want):
    return SPEC_TOL * max(1.0, float(np.abs(want).max()))


def synthetic_residuals(sc, B, seed):
    """Residuals at the scale the bench net produces (RMS ~1 cell on the centres,
    0.05 on response and attenuation), drawn directly so the oracle's CPU MLP is
    not needed for 300 positions; the MLP is checked on its own below."""
    rng = np.random.default_rng(seed)
    cel = (np.pi / 2) / sc.H
    n = sc.n
    return swr.Residuals(rng.normal(0, cel, (B, n, 2)).astype(np.float32),
                         rng.normal(0, 0.05, (B, n, 2)).astype(np.float32),
                         rng.normal(0, 0.05, (B, n)).astype(np.float32))


@pytest.fixture(scope="module", params=[10000, 50000], ids=["n10k", "n50k"])
def big(request):
    n = request.param
    sc = make_scene(n, seed=40 + n // 10000)
    sc.rssi_cal = (12.5, -61.0)
    ck = swr.Checkpoint.from_scene(sc)
    if n == 10000:
        ck.set_option("chunk", 128)    # the default (1024) would hold all 300 positions in one chunk
    assert int(ck.get_option("chunk")) < B
    return sc, ck, O.Port(sc)


def _res_b(res, b):
    return (res.d_center[b], res.d_response[b], res.d_atten[b])


def test_setup_bit_exact_at_size(big):
    sc, ck, port = big
    res = synthetic_residuals(sc, 3, seed=1)
    got = swr.setup(ck, res)
    for b in range(3):
        want = port.prepare(_res_b(res, b))
        np.testing.assert_array_equal(got["state"][b], want["state"])
        np.testing.assert_array_equal(got["rows"][b], want["rows"])
        np.testing.assert_array_equal(got["cols"][b], want["cols"])
        assert int(got["tile_count"][b].sum()) == int(want["tile_offset"][-1])


def test_bins_and_spectra_at_size(big):
    sc, ck, port = big
    res = synthetic_residuals(sc, B, seed=2)
    bins = swr.bins(ck, res)
    step = 1 if sc.n <= 10000 else 3
    for b in range(0, B, step):
        want = port.prepare(_res_b(res, b))
        np.testing.assert_array_equal(bins[b][0], want["tile_offset"])
        np.testing.assert_array_equal(bins[b][1], want["tile_prims"])
    spectra = swr.rasterize(ck, res)
    chunk = int(ck.get_option("chunk"))
    sample = sorted(b for b in {0, 1, chunk - 1, chunk, chunk + 1, 2 * chunk - 1, 2 * chunk, B - 2, B - 1}
                    | set(range(5, B, 37)) if b < B)
    for b in sample:
        want = port.rasterize(_res_b(res, b), precise=True)
        assert np.abs(spectra[b] - want).max() <= spec_tol(want), b
    # the heads on these spectra agree exactly with the oracle's heads on them
    pooled, rc, _ = swr.heads(ck, spectra[sample])
    for k, b in enumerate(sample):
        assert tuple(rc[k]) == port.aoa(spectra[b])[:2]
        assert pooled[k] == pytest.approx(port.pooled(spectra[b]), rel=1e-12)


@pytest.mark.parametrize("precision", [swr.MLP_FP16X3, swr.MLP_FP32], ids=["fp16x3", "fp32"])
def test_mlp_at_size(big, precision):
    sc, ck, port = big
    ck.set_option("mlp_precision", precision)
    pos = random_positions(B, seed=3)
    p01 = swr.normalize_position(ck, pos)
    res = swr.predict_residuals(ck, p01)
    for b in (0, 157, B - 1):
        want = port.predict(p01[b], precise=True)
        for g, w in zip(_res_b(res, b), want):
            assert np.abs(g - w).max() <= 2e-6 * max(1.0, float(np.abs(w).max()))


def test_render_at_size_equals_raster_of_own_residuals(big):
    """The chunked render pipeline (MLP -> setup -> bins -> raster -> heads, two
    device chunks, D2H overlapped) returns exactly rasterize() of the residuals it
    predicts; a sample is also checked against the oracle and its heads."""
    sc, ck, port = big
    ck.set_option("mlp_precision", swr.MLP_FP16X3)
    pos = random_positions(B, seed=4)
    out = swr.render(ck, pos, rssi=True)
    p01 = swr.normalize_position(ck, pos)
    res = swr.predict_residuals(ck, p01)
    ras = swr.rasterize(ck, res)
    assert np.array_equal(out["spectra"], ras)
    for b in (0, 127, 128, 255, 256, B - 1):
        want = port.rasterize(_res_b(res, b), precise=True)
        assert np.abs(out["spectra"][b] - want).max() <= spec_tol(want), b
        assert out["pooled"][b] == pytest.approx(port.pooled(want), rel=1e-5)
        r, c, el, az = port.aoa(want)
        if tuple(out["aoa_rc"][b]) != (r, c):
            mag = np.hypot(want[..., 0].astype(np.float64), want[..., 1])
            top = np.sort(mag.ravel())[-2:]
            assert top[1] - top[0] <= spec_tol(want)
    slope, intercept = ck.get_option("rssi_slope"), ck.get_option("rssi_intercept")
    np.testing.assert_allclose(out["rssi"], slope * out["pooled"] + intercept, rtol=0, atol=1e-12)
