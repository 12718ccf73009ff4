"""The ``upsample`` CLI on the GPU (gf/cli.py:72-101): its output files are
the REAL reference CLI's, byte for byte, on the fixtures under
tests/golden/io (make_golden_io.py); image bytes are converted on the device
(gf_image_unpack_u8 / gf_image_pack_u8); exit codes as the reference; the
DGFT checkpoint of ``train-toy`` loads back."""

import os
import shutil

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

IO = os.path.join(os.path.dirname(__file__), "golden", "io")


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


@pytest.fixture
def io_dir(tmp_path):
    for f in os.listdir(IO):
        shutil.copy(os.path.join(IO, f), tmp_path / f)
    return tmp_path


RUNS = [("out_joint.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm"]),
        ("out_joint_r2.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm",
                              "--radius", "2", "--eps", "1e-3"]),
        ("out_highres.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm",
                             "--variant", "highres", "--radius", "3", "--eps", "1e-2"]),
        ("out_gray.pgm", ["--guide", "guide1.pgm", "--low-res-output", "low1.pgm"]),
        ("out_png.png", ["--guide", "guide.png", "--low-res-output", "low.png"])]


@pytest.mark.parametrize("name,argv", RUNS)
def test_upsample_reproduces_reference_cli_bytes(gfb, io_dir, name, argv):
    from paper_1803_05619_b200 import cli, fileio

    cwd = os.getcwd()
    os.chdir(io_dir)
    try:
        assert cli.main(["upsample", *argv, "--out", name]) == 0
        got = fileio.read_png_bytes(name) if name.endswith(".png") else fileio.read_ppm_bytes(name)
        ref = "ref_" + name
        want = fileio.read_png_bytes(ref) if name.endswith(".png") else fileio.read_ppm_bytes(ref)
        assert np.array_equal(got, want)
        # fp32 production kernels: within one 8-bit level of the reference
        assert cli.main(["upsample", *argv, "--dtype", "f32", "--out", "f32_" + name]) == 0
        got32 = (fileio.read_png_bytes if name.endswith(".png") else fileio.read_ppm_bytes)(
            "f32_" + name)
        assert np.abs(got32.astype(int) - want.astype(int)).max() <= 1
    finally:
        os.chdir(cwd)


def test_upsample_exit_codes(gfb, io_dir, capsys):
    from paper_1803_05619_b200 import cli

    cwd = os.getcwd()
    os.chdir(io_dir)
    try:
        assert cli.main(["upsample", "--guide", "guide.ppm", "--low-res-output", "low1.pgm",
                         "--out", "x.ppm"]) == 3  # channel mismatch
        assert cli.main(["upsample", "--guide", "missing.ppm", "--low-res-output", "low.ppm",
                         "--out", "x.ppm"]) == 2
        open("bad.ppm", "wb").write(b"P6\n4 4\n255\n")
        assert cli.main(["upsample", "--guide", "bad.ppm", "--low-res-output", "low.ppm",
                         "--out", "x.ppm"]) == 2
        assert cli.main(["upsample", "--guide", "guide.ppm", "--low-res-output", "low.ppm",
                         "--radius", "-1", "--out", "x.ppm"]) == 3
        assert "error" in capsys.readouterr().err
    finally:
        os.chdir(cwd)


def test_device_image_round_trip(gfb, io_dir):
    from paper_1803_05619_b200 import fileio

    for name in ("guide.ppm", "guide1.pgm", "guide.png"):
        t = fileio.read_image_device(io_dir / name)
        assert torch.equal(t[0].permute(1, 2, 0).cpu(),
                           torch.from_numpy(fileio.load_image(io_dir / name)))
        out = io_dir / ("rt_" + name)
        fileio.write_image_device(out, t)
        read = fileio.read_png_bytes if name.endswith(".png") else fileio.read_ppm_bytes
        assert np.array_equal(read(out), read(io_dir / name))


def test_checkpoint_reference_file_and_train_toy(gfb, io_dir, capsys):
    from paper_1803_05619_b200 import cli

    model = gfb.build_model(seed=3)
    gfb.load_checkpoint(model, io_dir / "ref_model.dgft")  # written by the reference
    gfb.save_checkpoint(model, io_dir / "mine.dgft")
    assert (io_dir / "mine.dgft").read_bytes() == (io_dir / "ref_model.dgft").read_bytes()
    rc = cli.main(["train-toy", "--task", "affine", "--steps", "3", "--checkpoint",
                   str(io_dir / "toy.dgft")])
    assert rc in (0, 1)  # 3 steps need not improve 10x
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "step,loss" and len(lines) == 5
    m2 = gfb.build_model(seed=0)
    gfb.load_checkpoint(m2, io_dir / "toy.dgft")
