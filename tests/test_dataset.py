"""Dataset I/O: manifest.json + spectra.bin read
through the C ABI against the reference's own load_dataset on datasets the
reference simulates and saves itself (oracle/_ref: wavesim + dataset.cpp), and
the batched train::evaluate over a split against the reference's."""
import os
import shutil

import numpy as np
import pytest

import oracle as O
from paper_2506_12787_b200 import swr
from paper_2506_12787_b200.scene import make_scene

H, W = 30, 60


@pytest.fixture(scope="module")
def ds_dir(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("ds"))
    h, bbox = O.make_dataset(d, H, W, 40, 11)
    return d, h, bbox


def test_reader_matches_reference_load(ds_dir):
    d, h, bbox = ds_dir
    ds = swr.Dataset(d)
    rh, rpos, rspec = O.load_dataset(d, H, W)
    assert ds.manifest_hash == h == rh
    assert (ds.H, ds.W, ds.samples) == (H, W, len(rpos))
    np.testing.assert_array_equal(ds.bbox, bbox)
    pos, spec = ds.read()
    np.testing.assert_array_equal(pos, rpos)
    np.testing.assert_array_equal(spec, rspec)
    # split rule (wavesim.hpp:152-154): original index % 10 == 0 -> test; indices are post-exclusion
    tr, te, al = ds.split(ds.TRAIN), ds.split(ds.TEST), ds.split(ds.ALL)
    assert len(tr) + len(te) == ds.samples and np.array_equal(al, np.arange(ds.samples))
    p2, s2 = ds.read(te[::-1])
    np.testing.assert_array_equal(s2, rspec[te[::-1]])
    np.testing.assert_array_equal(p2, rpos[te[::-1]])


def test_reader_rejects_bad_files(ds_dir, tmp_path):
    d, _, _ = ds_dir
    bad = str(tmp_path / "bad")
    shutil.copytree(d, bad)
    with open(os.path.join(bad, "spectra.bin"), "ab") as fh:
        fh.write(b"\0")
    with pytest.raises(swr.SwrError, match="trailing bytes"):
        swr.Dataset(bad)
    with open(os.path.join(bad, "spectra.bin"), "r+b") as fh:
        fh.truncate(os.path.getsize(os.path.join(d, "spectra.bin")) - 4)
    with pytest.raises(swr.SwrError, match="unexpected end of file"):
        swr.Dataset(bad)
    with open(os.path.join(bad, "manifest.json"), "w") as fh:
        fh.write('{"format": "something-else", "version": 1}')
    with pytest.raises(swr.SwrError, match="not a version-1 dataset manifest"):
        swr.Dataset(bad)
    ds = swr.Dataset(d)
    with pytest.raises(ValueError):
        ds.read([ds.samples])


def _bound_scene(bbox):
    sc = make_scene(300, seed=3, H=H, W=W)
    sc.bbox_min, sc.bbox_max = tuple(bbox[:3]), tuple(bbox[3:])
    return sc


@pytest.mark.gpu
@pytest.mark.parametrize("split", [0, 1, 2])
def test_evaluate_dataset_matches_reference(ds_dir, split):
    d, h, bbox = ds_dir
    sc = _bound_scene(bbox)
    ref = O.Reference(sc)
    ref.set_dataset(h, bbox)
    want = ref.evaluate(d, split)
    ck = swr.Checkpoint.from_scene(sc)
    ck.set_option("mlp_precision", swr.MLP_FP32)
    ck.set_manifest_hash(h)
    ds = swr.Dataset(d)
    got = swr.evaluate_dataset(ck, ds, split)
    np.testing.assert_array_equal(got["sample_id"], want[:, 0].astype(np.int32))
    assert np.abs(got["psnr"] - want[:, 1]).max() <= 1e-4
    assert np.abs(got["ssim"] - want[:, 2]).max() <= 1e-6
    assert (np.abs(got["l1"] - want[:, 3]) / np.abs(want[:, 3])).max() <= 1e-5


@pytest.mark.gpu
def test_evaluate_dataset_hash_mismatch(ds_dir):
    d, h, bbox = ds_dir
    ck = swr.Checkpoint.from_scene(_bound_scene(bbox))
    ck.set_manifest_hash(h ^ 1)
    with pytest.raises(swr.SwrError, match="different dataset"):
        swr.evaluate_dataset(ck, swr.Dataset(d), 1)
