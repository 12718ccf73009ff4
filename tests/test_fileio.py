"""File formats of the reference (gf/fileio.py) -- host I/O, no GPU: the DGFT
container and PPM/PGM/PNG byte conventions, pinned by files the REAL
reference wrote (tests/golden/io, make_golden_io.py)."""

import os

import numpy as np
import pytest

from paper_1803_05619_b200 import fileio

IO = os.path.join(os.path.dirname(__file__), "golden", "io")


def test_dgft_reads_reference_file_and_writes_identical_bytes(tmp_path):
    got = fileio.load_tensors(os.path.join(IO, "ref.dgft"))
    vals = np.load(os.path.join(IO, "ref_dgft_values.npz"))
    assert list(got) == ["a", "bias", "ünï"]
    for k, v in zip(got, (vals["t0"], vals["t1"], vals["t2"])):
        assert np.array_equal(got[k], v)
    out = tmp_path / "x.dgft"
    fileio.save_tensors(out, got)
    assert out.read_bytes() == open(os.path.join(IO, "ref.dgft"), "rb").read()


def test_dgft_errors(tmp_path):
    good = open(os.path.join(IO, "ref.dgft"), "rb").read()
    for bad, what in ((b"XXXX" + good[4:], "magic"), (good[:4] + b"\x02" + good[5:], "version"),
                      (good[:-3], "truncated"), (good + b"\0", "trailing")):
        p = tmp_path / f"{what}.dgft"
        p.write_bytes(bad)
        with pytest.raises(fileio.ImageFormatError):
            fileio.load_tensors(p)
    with pytest.raises(ValueError):
        fileio.save_tensors(tmp_path / "n.dgft", {"x": np.full((1, 1, 1), np.nan)})
    with pytest.raises(ValueError):
        fileio.save_tensors(tmp_path / "n.dgft", {"x": np.zeros((2, 2))})


@pytest.mark.parametrize("name", ["guide.ppm", "low.ppm", "guide1.pgm", "guide.png"])
def test_image_round_trip_is_byte_exact(tmp_path, name):
    img = fileio.load_image(os.path.join(IO, name))
    assert img.dtype == np.float64 and img.min() >= 0 and img.max() <= 1
    out = tmp_path / ("o" + os.path.splitext(name)[1])
    fileio.save_image(out, img)
    if name.endswith(".png"):
        assert np.array_equal(fileio.load_image(out), img)
    else:
        assert out.read_bytes() == open(os.path.join(IO, name), "rb").read()


def test_ppm_header_comments_and_errors(tmp_path):
    px = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    p = tmp_path / "c.ppm"
    p.write_bytes(b"P6 # comment\n3 # w\n 2\n255\n" + px.tobytes())
    assert np.array_equal(fileio.read_ppm_bytes(p), px)
    assert np.array_equal(fileio.load_ppm(p), px / 255.0)
    for data in (b"P3\n3 2\n255\n" + px.tobytes(), b"P6\n3 2\n65535\n" + px.tobytes(),
                 b"P6\n3 2\n255\n" + px.tobytes()[:-1], b"P6\n3", b"P6\n0 2\n255\n"):
        p.write_bytes(data)
        with pytest.raises(fileio.ImageFormatError):
            fileio.load_ppm(p)
    with pytest.raises(ValueError):
        fileio.save_ppm(tmp_path / "x.ppm", np.zeros((2, 2, 2)))


def test_save_clamps_and_rounds_half_to_even(tmp_path):
    img = np.array([[[-0.5, 0.5 / 255.0, 1.5 / 255.0], [2.5 / 255.0, 1.2, 0.2]]])
    fileio.save_ppm(tmp_path / "r.ppm", img)
    assert list(fileio.read_ppm_bytes(tmp_path / "r.ppm").reshape(-1)) == [0, 0, 2, 2, 255, 51]
