"""Record loader (data::load_records, dataset.cpp:65-99) on the GPU:
planar CHW records -> HWC rows + labels, equal to the oracle restatement,
with the reference's error messages (cf. test_dataset.cpp:53-98)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write(tmp_path, n, h, w, c, n_classes, seed=0, name="rec.bin"):
    rng = np.random.default_rng(seed)
    rec = np.empty((n, 1 + h * w * c), np.uint8)
    rec[:, 0] = rng.integers(0, n_classes, n)
    rec[:, 1:] = rng.integers(0, 256, (n, h * w * c))
    p = tmp_path / name
    p.write_bytes(rec.tobytes())
    return p, rec.tobytes()


@pytest.mark.parametrize("h,w,c,n", [(32, 32, 3, 500), (2, 2, 3, 7), (5, 3, 1, 11), (224, 224, 3, 3),
                                          (299, 299, 3, 5), (17, 13, 40000, 2)])
def test_records_vs_oracle(pkg, oracle_mod, torch_cuda, tmp_path, h, w, c, n):
    C = pkg.codec
    path, raw = _write(tmp_path, n, h, w, c, 10)
    px, lab = C.load_records_dev(str(path), C.ImageShape(h, w, c), 10, max_records=n)
    want_px, want_lab = oracle_mod.records_to_hwc(raw, h, w, c)
    assert np.array_equal(px.cpu().numpy(), want_px)
    assert np.array_equal(lab.cpu().numpy(), want_lab)


def test_records_errors(pkg, torch_cuda, tmp_path):
    C, E = pkg.codec, pkg.errors
    shape = C.ImageShape(2, 2, 3)
    path, raw = _write(tmp_path, 4, 2, 2, 3, 10)
    with pytest.raises(E.FormatError, match=r"^records: label \d+ outside 3 classes in "):
        C.load_records_dev(str(path), shape, 3, max_records=4)
    (tmp_path / "part.bin").write_bytes(raw[:-2])
    with pytest.raises(E.FormatError, match="trailing partial record"):
        C.load_records_dev(str(tmp_path / "part.bin"), shape, 10, max_records=4)
    (tmp_path / "empty.bin").write_bytes(b"")
    with pytest.raises(E.FormatError, match="no records in"):
        C.load_records_dev(str(tmp_path / "empty.bin"), shape, 10, max_records=4)
    with pytest.raises(E.FormatError, match="cannot open"):
        C.load_records_dev(str(tmp_path / "nope.bin"), shape, 10, max_records=4)
    with pytest.raises(E.ShapeError, match="extents must be positive"):
        C.load_records_dev(str(path), C.ImageShape(0, 2, 3), 10, max_records=4)


def test_records_large_label_error(pkg, torch_cuda, tmp_path):
    """Records past the whole-record staging budget take the tiled kernel;
    its label check names the first offending record like the staged one."""
    C, E = pkg.codec, pkg.errors
    path, raw = _write(tmp_path, 6, 299, 299, 3, 10, seed=3)
    with pytest.raises(E.FormatError, match=r"^records: label \d+ outside 2 classes in "):
        C.load_records_dev(str(path), C.ImageShape(299, 299, 3), 2, max_records=6)
