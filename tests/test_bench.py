"""The bench contract (bench.py): one JSON line with the driver's keys, the
roofline / cpu_baseline / e2e / clocks / gpu_launches records and the post-timing
parity check of the timed batch; the reference arm on the host cores."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_ref

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not has_ref(), reason="reference build absent")
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--n", "1500", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference" and d["metric"] == "spectra/sec" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_native_line_carries_the_contract():
    d = _run(["--n", "3000", "--batch", "96", "--steps", "3", "--warmup", "3", "--no-spec-sized"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "parity_ok"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == 96 * (90 * 360 * 8 + 40)
    r = d["roofline"]
    assert 0 < r["frac"] < 1 and r["bound"] == "tensor" and r["kernel"] == "deform MLP (mlp_tc2_kernel)"
    assert d["parity_ok"] is True and d["parity"]["aoa_ok"] is True
    assert d["cpu_baseline"] is None or d["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.skipif(not has_ref(), reason="reference build absent")
def test_parity_check_is_not_vacuous():
    """bench.parity_check (the post-timing check behind parity_ok) passes the GPU's own
    outputs and fails each kind of corruption: one cell off by 1e-4 of the peak, the
    pooled magnitude off by 1e-4 relative, the AoA moved to a non-tied cell."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from paper_2506_12787_b200 import swr
    from paper_2506_12787_b200.scene import make_scene, random_positions
    sc = make_scene(1500, seed=4)
    ck = swr.Checkpoint.from_scene(sc)
    pos = random_positions(4, seed=8)
    out = swr.render(ck, pos)
    idx = np.arange(4)
    args = (ck, sc, pos, idx)
    good = bench.parity_check(*args, out["spectra"].copy(), out["pooled"].copy(), out["aoa_rc"].copy())
    assert good["ok"], good
    spec = out["spectra"].copy()
    spec[1, 40, 100, 0] += 1e-4 * max(1.0, float(np.abs(spec[1]).max()))
    assert not bench.parity_check(*args, spec, out["pooled"], out["aoa_rc"])["ok"]
    pooled = out["pooled"].copy()
    pooled[2] *= 1 + 1e-4
    assert not bench.parity_check(*args, out["spectra"], pooled, out["aoa_rc"])["ok"]
    rc = out["aoa_rc"].copy()
    mag = np.hypot(out["spectra"][3][..., 0].astype(np.float64), out["spectra"][3][..., 1])
    r, c = np.unravel_index(int(np.argmin(mag)), mag.shape)     # the weakest cell: no tie with the peak
    rc[3] = (r, c)
    assert not bench.parity_check(*args, out["spectra"], out["pooled"], rc)["ok"]
