"""Width-512 deformation MLP on tcgen05 (k_mlp_wide.cu; BASELINE config 5's "wide"
net, TrainConfig.width up to 512, training.hpp:100): residuals within the FP32 bar
of the FP64 oracle (deform.cpp:140-207 restated), the same bar as the FP32
CUDA-core kernel, across several layer-GEMM row blocks (the last one padded),
and the render from those residuals equal to the oracle's rasterize()."""
import numpy as np
import pytest

import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene, random_positions

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[(700, 512), (333, 300)], ids=["w512", "w300"])
def wide(request):
    n, width = request.param
    sc = make_scene(n, seed=51, width=width)
    return sc, O.Port(sc)


@pytest.mark.parametrize("block_rows", [None, 512])
def test_wide_mlp_residuals_fp32_grade(wide, block_rows):
    sc, port = wide
    ck = swr.Checkpoint.from_scene(sc)
    assert ck.get_option("mlp_precision") == swr.MLP_FP16X3      # the tensor-core path is the default
    if block_rows:
        ck.set_option("wide_block_rows", block_rows)             # several row blocks, the last one padded
    ck32 = swr.Checkpoint.from_scene(sc)
    ck32.set_option("mlp_precision", swr.MLP_FP32)
    pos = random_positions(6, seed=8)
    p01 = swr.normalize_position(ck, pos)
    r16 = swr.predict_residuals(ck, p01)
    r32 = swr.predict_residuals(ck32, p01)
    worst = 0.0
    for b in (0, 3, 5):
        want = port.predict(p01[b], precise=True)
        for g16, g32, w in zip((r16.d_center[b], r16.d_response[b], r16.d_atten[b]),
                               (r32.d_center[b], r32.d_response[b], r32.d_atten[b]), want):
            bar = 2e-6 * max(1.0, float(np.abs(w).max()))
            assert np.abs(g32 - w).max() <= bar
            worst = max(worst, float(np.abs(g16 - w).max()) / bar)
    assert worst <= 1.0, worst
    assert ck.get_option("mlp_reruns") == 0


def test_wide_render_from_own_residuals(wide):
    sc, port = wide
    ck = swr.Checkpoint.from_scene(sc)
    pos = random_positions(4, seed=9)
    out = swr.render(ck, pos)
    p01 = swr.normalize_position(ck, pos)
    res = swr.predict_residuals(ck, p01)
    for b in range(4):
        want = port.rasterize((res.d_center[b], res.d_response[b], res.d_atten[b]), precise=True)
        assert np.abs(out["spectra"][b] - want).max() <= 1e-5 * max(1.0, float(np.abs(want).max()))
