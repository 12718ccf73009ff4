"""Fixtures of the reference's file formats and its upsample CLI.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_io.py

Writes small files under tests/golden/io/ with the REAL reference
(gf/fileio.py, gf/cli.py, gf/training.py): a DGFT container, a checkpoint of
build_model(seed=3), PPM / PGM / PNG inputs and the reference CLI's
``upsample`` outputs for them (joint and highres variants).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
sys.path.insert(0, REF)

from guidedfilter import cli, fileio, training  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(77)
    tensors = {"a": rng.standard_normal((3, 4, 2)), "bias": rng.uniform(-1, 1, (1, 1, 5)),
               "ünï": np.full((1, 2, 1), 0.125)}
    fileio.save_tensors(os.path.join(OUT, "ref.dgft"), tensors)
    np.savez(os.path.join(OUT, "ref_dgft_values.npz"), **{f"t{i}": v for i, v in
                                                          enumerate(tensors.values())})
    model = training.build_model(seed=3)
    training.save_checkpoint(model, os.path.join(OUT, "ref_model.dgft"))
    # images: smooth-ish guide and a low-res result, as 8-bit files
    imgs = training.synthetic_images(1, 48, 64, 3, seed=5)[0]
    low = training.bilinear_resize(np.clip(1.2 * imgs - 0.1, 0, 1), 12, 16)
    fileio.save_ppm(os.path.join(OUT, "guide.ppm"), imgs)
    fileio.save_ppm(os.path.join(OUT, "low.ppm"), low)
    fileio.save_ppm(os.path.join(OUT, "guide1.pgm"), imgs[:, :, :1])
    fileio.save_ppm(os.path.join(OUT, "low1.pgm"), low[:, :, :1])
    fileio.save_png(os.path.join(OUT, "guide.png"), imgs)
    fileio.save_png(os.path.join(OUT, "low.png"), low)
    runs = [("out_joint.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm"]),
            ("out_joint_r2.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm",
                                  "--radius", "2", "--eps", "1e-3"]),
            ("out_highres.ppm", ["--guide", "guide.ppm", "--low-res-output", "low.ppm",
                                 "--variant", "highres", "--radius", "3", "--eps", "1e-2"]),
            ("out_gray.pgm", ["--guide", "guide1.pgm", "--low-res-output", "low1.pgm"]),
            ("out_png.png", ["--guide", "guide.png", "--low-res-output", "low.png"])]
    cwd = os.getcwd()
    os.chdir(OUT)
    try:
        for name, argv in runs:
            rc = cli.main(["upsample", *argv, "--out", "ref_" + name])
            assert rc == 0, (name, rc)
    finally:
        os.chdir(cwd)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
