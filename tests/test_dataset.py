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


# ---------------------------------------------------------------- writer (save_dataset)

def _files(d):
    with open(os.path.join(d, "manifest.json"), "rb") as a, open(os.path.join(d, "spectra.bin"), "rb") as b:
        return a.read(), b.read()


def test_writer_round_trip_byte_identical(ds_dir, tmp_path):
    """A dataset the reference simulated and saved (save_dataset, dataset.cpp:183-203),
    read back and written again through the C ABI writer: manifest.json and
    spectra.bin are byte-identical, and so is the manifest fingerprint."""
    d, h, _ = ds_dir
    ds = swr.Dataset(d)
    meta = ds.meta()
    assert meta.mode in (b"tx_moving", b"rx_moving")
    pos, spec = ds.read()
    out = str(tmp_path / "one_call")
    assert swr.save_dataset(out, meta, pos, spec) == h
    assert _files(out) == _files(d)
    assert meta.manifest(ds.samples) == (_files(d)[0], h)
    # streamed in uneven chunks
    out2 = str(tmp_path / "stream")
    w = swr.DatasetWriter(out2, ds.H, ds.W)
    for a, b in [(0, 7), (7, 8), (8, 23), (23, ds.samples)]:
        w.append(pos[a:b], spec[a:b])
    assert w.close(meta) == h
    assert _files(out2) == _files(d)


def test_reference_loads_written_dataset(ds_dir, tmp_path):
    """The reference's own load_dataset reads what the writer wrote (a new manifest:
    other splits, normalisation, bbox, RSSI labels), with the same fingerprint."""
    d, _, _ = ds_dir
    ds = swr.Dataset(d)
    pos, spec = ds.read()
    n = 12
    rng = np.random.default_rng(5)
    meta = swr.DatasetMeta.build(H, W, mode="rx_moving", seed=77, normalization=0.123456789012345,
                                 train=[i for i in range(n) if i % 3], test=[i for i in range(n) if not i % 3],
                                 excluded=[4, 19], bbox_min=(0.31, 0.3, 0.29), bbox_max=(3.7, 2.71, 2.2),
                                 rssi_dbm=rng.normal(-60, 5, n), room=(5.0, 4.0, 3.0), reflectivity=0.35,
                                 max_bounces=2, fixed_node=(1.0, 2.0, 1.5), k_elements=8, spacing=0.05,
                                 wavelength=0.1)
    out = str(tmp_path / "new")
    hw = swr.save_dataset(out, meta, pos[:n], spec[:n])
    rh, rpos, rspec = O.load_dataset(out, H, W)
    assert rh == hw
    np.testing.assert_array_equal(rpos, pos[:n])
    np.testing.assert_array_equal(rspec, spec[:n])
    back = swr.Dataset(out)
    m2 = back.meta()
    assert (m2.mode, m2.seed, m2.max_bounces, m2.k_elements) == (b"rx_moving", 77, 2, 8)
    assert m2.manifest(n)[1] == hw


def test_writer_errors(tmp_path):
    meta = swr.DatasetMeta.build(H, W, mode="sideways")
    with pytest.raises(ValueError, match="unknown mobility mode"):
        meta.manifest(0)
    w = swr.DatasetWriter(str(tmp_path / "g"), H, W)
    with pytest.raises(ValueError, match="grid differs"):
        w.close(swr.DatasetMeta.build(H + 1, W))
    with pytest.raises(ValueError):
        swr.DatasetWriter(str(tmp_path / "z"), 0, W)


@pytest.mark.gpu
def test_writer_render_equals_render(ds_dir, tmp_path):
    """Rendered straight into a dataset on the GPU (chunked, file writes overlapped):
    the records equal swr.render of the same positions bit for bit, and the
    reference's load_dataset reads the directory."""
    d, h, bbox = ds_dir
    sc = _bound_scene(bbox)
    ck = swr.Checkpoint.from_scene(sc)
    rng = np.random.default_rng(3)
    pos = swr_positions = (bbox[:3] + rng.random((600, 3)) * (bbox[3:] - bbox[:3])).astype(np.float32)
    out = str(tmp_path / "rendered")
    w = swr.DatasetWriter(out, H, W)
    w.render(ck, pos)          # 600 positions: three 256-position chunks, the file writes overlapped
    meta = swr.DatasetMeta.build(H, W, train=list(range(600)), bbox_min=bbox[:3], bbox_max=bbox[3:])
    hw = w.close(meta)
    want = swr.render(ck, swr_positions)["spectra"]
    back = swr.Dataset(out)
    p2, s2 = back.read()
    np.testing.assert_array_equal(p2, pos)
    np.testing.assert_array_equal(s2, want)
    rh, _, rspec = O.load_dataset(out, H, W)
    assert rh == hw
    np.testing.assert_array_equal(rspec, want)
