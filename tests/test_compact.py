"""MEGS2 compact files (io.py) against files written and read by the
reference (tests/golden/compact.npz, make_golden.py gen_compact); the format
checks mirror the reference's test_io.py:96-145."""

from pathlib import Path

import numpy as np
import pytest

from paper_2509_07021_b200 import io as IO

GOLDEN = Path(__file__).resolve().parent / "golden"


def _golden():
    d = np.load(GOLDEN / "compact.npz")
    return d, d["raw"].tobytes()


def test_writer_is_byte_identical_to_reference():
    d, raw = _golden()
    data = IO.write_compact(d["position"], d["quat"], d["scale"], d["opacity"], d["diffuse"],
                            d["axis_raw"], d["sharpness"], d["amplitude"], d["n_lobes"])
    assert data == raw


def test_index_offsets_and_lobe_count():
    d, raw = _golden()
    offs, ml = IO.compact_index(raw)
    assert ml == 5 and offs.size == d["n_lobes"].size + 1
    sizes = 57 + 28 * d["n_lobes"]
    assert np.array_equal(np.diff(offs.astype(np.int64)), sizes)
    assert int(offs[0]) == 12 and int(offs[-1]) == len(raw)


def test_empty_file_and_format_errors():
    empty = IO.write_compact(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                             np.zeros((0, 3)), np.zeros((0, 3, 3)), np.zeros((0, 3)), np.zeros((0, 3, 3)),
                             np.zeros(0, int))
    assert empty == b"MEGS2\x00" + b"\x01\x00" + b"\x00\x00\x00\x00"
    offs, ml = IO.compact_index(empty)
    assert offs.tolist() == [12] and ml == 0
    _, raw = _golden()
    bad = bytearray(raw)
    bad[0] = 0x58
    with pytest.raises(IO.SceneFormatError):
        IO.compact_index(bytes(bad))
    bad = bytearray(raw)
    bad[6] = 2
    with pytest.raises(IO.SceneFormatError):
        IO.compact_index(bytes(bad))
    with pytest.raises(IO.TruncatedFileError):
        IO.compact_index(raw[:-3])
    with pytest.raises(IO.TruncatedFileError):
        IO.compact_index(raw[:9])
    with pytest.raises(IO.SceneFormatError):
        IO.compact_index(raw + b"\x00")


@pytest.mark.gpu
def test_gpu_decode_matches_reference_scene_params():
    import torch
    d, raw = _golden()
    g = IO.load_compact(raw)
    torch.cuda.synchronize()
    for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness", "amplitude"):
        got = getattr(g, f).cpu().numpy()
        want = np.asarray(d[f], np.float64).astype(np.float32)
        assert np.array_equal(got, want), f
    assert np.array_equal(g.lobe_mask.cpu().numpy(), d["lobe_mask"].astype(np.float32))


@pytest.mark.gpu
def test_loaded_scene_renders_like_uploaded_arrays():
    import torch
    from paper_2509_07021_b200.camera import Camera
    from paper_2509_07021_b200.rasterizer import GaussianTensors, Rasterizer

    d, raw = _golden()

    class P:
        pass
    p = P()
    for f in ("position", "quat", "log_scale", "opacity", "diffuse", "axis_raw", "sharpness", "amplitude",
              "lobe_mask"):
        setattr(p, f, d[f])
    cam = Camera.look_at((0.0, -3.0, 0.5), (0, 0, 0), width=96, height=80, fx=90)
    rast = Rasterizer()
    a = rast.forward(IO.load_compact(raw), cam).img.clone()
    b = rast.forward(GaussianTensors.from_arrays(p), cam).img
    assert torch.equal(a, b) and float(a.abs().max()) > 0
