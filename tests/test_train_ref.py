"""CPU tests of the training oracle: the reference's own train::train
(training.cpp:198-376, compiled from its sources into oracle/_ref) with the
Eigen-free deform_backward restatement (oracle/ref_shim/deform_restated.cpp)
pinned by finite differences, and the reference's training tests restated
(test_training.cpp:228-322) on a dataset simulated by the reference itself."""
import csv
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import has_ref
import oracle as O
from paper_2506_12787_b200.scene import make_scene

pytestmark = pytest.mark.skipif(not has_ref(), reason="reference build absent (GPU box)")


def tiny_cfg(**kw):
    """tiny_config() of test_training.cpp:55-63 on the TrainConfig defaults (training.hpp:96-112)."""
    c = dict(primitives=6, bands_center=10, bands_position=6, width=156, cutoff_radius=3.0, tile=16,
             lr_gaussian=1e-2, lr_mlp=8e-3, lambda1=0.7, coarse_iters=12, fine_iters=8, anneal_scale=1.0,
             anneal_threshold=5, seed=99)
    c.update(kw)
    return SimpleNamespace(**c)


@pytest.fixture(scope="module")
def tiny_ds(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("tiny_ds"))
    O.make_dataset(d, 12, 16, 8, 5)
    return d


def test_deform_backward_restatement_matches_finite_differences():
    sc = make_scene(12, seed=4, H=16, W=32, width=24)
    ref = O.Reference(scene=sc)
    rng = np.random.default_rng(1)
    pos01 = np.array([0.3, 0.6, 0.45], np.float32)
    n = sc.n
    up = (rng.standard_normal((n, 2)).astype(np.float32), rng.standard_normal((n, 2)).astype(np.float32),
          rng.standard_normal(n).astype(np.float32))
    gw, gb = ref.deform_backward(pos01, up)

    def loss(weights, biases):
        s2 = make_scene(12, seed=4, H=16, W=32, width=24)
        s2.weights, s2.biases = weights, biases
        dc, dr, da = O.Reference(scene=s2).predict(pos01)
        return float(np.sum(up[0] * dc, dtype=np.float64) + np.sum(up[1] * dr, dtype=np.float64)
                     + np.sum(up[2] * da, dtype=np.float64))

    bad = 0
    checks = 0
    for layer in (0, 2, 5, 7, 8, 9, 10):
        for _ in range(3):
            r = rng.integers(sc.weights[layer].shape[0])
            c = rng.integers(sc.weights[layer].shape[1])
            eps = 1e-2 * max(1e-2, abs(float(sc.weights[layer][r, c])))
            wp = [w.copy() for w in sc.weights]
            wm = [w.copy() for w in sc.weights]
            wp[layer][r, c] += eps
            wm[layer][r, c] -= eps
            fd = (loss(wp, sc.biases) - loss(wm, sc.biases)) / (2 * eps)
            an = float(gw[layer][r, c])
            checks += 1
            if abs(fd - an) > 2e-2 * max(abs(fd), abs(an)) + 1e-3:
                bad += 1
        bp = [b.copy() for b in sc.biases]
        bm = [b.copy() for b in sc.biases]
        bp[layer][0] += 1e-3
        bm[layer][0] -= 1e-3
        fd = (loss(sc.weights, bp) - loss(sc.weights, bm)) / 2e-3
        checks += 1
        if abs(fd - float(gb[layer][0])) > 2e-2 * max(abs(fd), abs(float(gb[layer][0]))) + 1e-3:
            bad += 1
    assert bad <= 1, f"{bad} of {checks} finite-difference checks failed"  # one ReLU kink crossing tolerated


def test_reference_training_is_reproducible_and_validates(tiny_ds):
    ref = O.Reference(scene=make_scene(4, seed=1, H=12, W=16, width=24))
    a = ref.train(tiny_ds, tiny_cfg())
    b = ref.train(tiny_ds, tiny_cfg())
    assert a.iteration() == 20
    for k in ("center_raw", "cholesky", "atten_logit", "response"):
        np.testing.assert_array_equal(getattr(a.sc, k), getattr(b.sc, k))
    for wa, wb in zip(a.sc.weights, b.sc.weights):
        np.testing.assert_array_equal(wa, wb)
    with pytest.raises(ValueError):
        ref.train(tiny_ds, tiny_cfg(lambda1=1.5))
    with pytest.raises(ValueError):
        ref.train(tiny_ds, tiny_cfg(coarse_iters=-1))


def test_reference_coarse_loss_decreases(tiny_ds, tmp_path):
    ref = O.Reference(scene=make_scene(4, seed=1, H=12, W=16, width=24))
    log = str(tmp_path / "log.csv")
    ref.train(tiny_ds, tiny_cfg(primitives=24, coarse_iters=150, fine_iters=0), log_path=log)
    rows = list(csv.reader(open(log)))
    assert rows[0] == ["iteration", "stage", "loss", "l1_term", "ssim_term", "wall_ms"]
    loss = np.array([float(r[2]) for r in rows[1:]])
    assert len(loss) == 150 and loss[:15].sum() > loss[-15:].sum()
