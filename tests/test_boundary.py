"""CPU-only checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/gf_b200.h declares, ctypes signatures cover the
header, and the host-side validation mirrors the reference's exceptions.
No compute calls are made (there is no GPU here)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gf_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("gf_", "gn_", "gnk_"))))


def test_header_declares_expected_entry_points():
    names = header_functions()
    for must in ("gf_joint_fwd", "gf_joint_bwd", "gf_highres_fwd", "gf_highres_bwd",
                 "gn_forward", "gn_backward", "gf_mean_filter", "gf_bilinear_resize_adjoint",
                 "gf_mse_loss", "gf_version"):
        assert must in names
    assert len(names) >= 19


def test_library_exports_every_header_symbol():
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), f"{name} not exported by {_lib.LIB_PATH}"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(header_functions())
    assert lib.gf_version() == 100


def test_library_is_built_for_sm100a():
    import subprocess

    from paper_1803_05619_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out


def test_params_validation_mirrors_reference():
    from paper_1803_05619_b200 import GuidedFilterParams

    with pytest.raises(ValueError):
        GuidedFilterParams(radius=-1)
    with pytest.raises(ValueError):
        GuidedFilterParams(radius=1, eps=-1e-3)
    with pytest.raises(ValueError):
        GuidedFilterParams(radius=1.5)
    with pytest.raises(ValueError):
        GuidedFilterParams(radius=1, eps=float("nan"))
    p = GuidedFilterParams()
    assert p.radius == 1 and p.eps == 1e-8


def test_input_validation_without_gpu():
    import torch

    from paper_1803_05619_b200._tensors import as_img

    with pytest.raises(ValueError):
        as_img(np.zeros((2, 2)), "x")                  # rank
    with pytest.raises(ValueError):
        as_img(np.zeros((0, 2, 1)), "x")               # empty dim
    with pytest.raises(ValueError):
        as_img(np.zeros((2, 2, 1), np.float32), "x")   # reference requires float64
    with pytest.raises(ValueError):
        as_img(torch.zeros(1, 1, 2, 2), "x")           # CPU tensor: no CPU fallback
    with pytest.raises(ValueError):
        as_img(torch.zeros(1, 1, 2, 2, dtype=torch.int32), "x")


def test_c_abi_argument_errors_without_gpu():
    """Shape/param errors are detected before any launch (ValueError codes)."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    # radius < 0
    rc = lib.gf_joint_fwd(0, 0, 0, 0, 0, 1, 3, 4, 4, 8, 8, -1, 1e-2, 0, 0, 0, 0)
    assert rc == _lib.GF_ERR_ARG and "radius" in _lib.last_error()
    # eps < 0
    rc = lib.gf_joint_fwd(0, 0, 0, 0, 0, 1, 3, 4, 4, 8, 8, 1, -1.0, 0, 0, 0, 0)
    assert rc == _lib.GF_ERR_ARG and "eps" in _lib.last_error()
    # guide_hi smaller than guide_lo (gf/guided.py:165-168)
    rc = lib.gf_joint_fwd(0, 0, 0, 0, 0, 1, 3, 8, 8, 4, 4, 1, 1e-2, 0, 0, 0, 0)
    assert rc == _lib.GF_ERR_ARG and "smaller" in _lib.last_error()
    # highres channel mismatch
    rc = lib.gf_highres_fwd(0, 0, 0, 0, 1, 2, 3, 8, 8, 1, 1e-2, 0, 0, 0, 0)
    assert rc == _lib.GF_ERR_ARG
    # dtype
    rc = lib.gf_mean_filter(7, 0, 0, 1, 4, 4, 1, 0)
    assert rc == _lib.GF_ERR_ARG
    # workspace too small (generic path needs workspace)
    rc = lib.gf_joint_fwd(1, 0, 0, 0, 0, 1, 3, 4, 5, 8, 10, 1, 1e-2, 0, 0, 0, 0)
    assert rc == _lib.GF_ERR_WORKSPACE
    # guidance limits
    rc = lib.gn_forward(0, 0, 0, 0, 1, 3, 3, 65, 4, 4, 0, 1 << 30, 0, 0)
    assert rc == _lib.GF_ERR_UNSUPPORTED


def test_workspace_queries_are_pure():
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    assert lib.gf_joint_workspace_bytes(1, 1, 3, 16, 16, 64, 64, 1) >= 17 * 3 * 256 * 8
    assert lib.gf_highres_workspace_bytes(1, 1, 1, 3, 32, 32, 2) >= 17 * 3 * 1024 * 8
    assert lib.gn_param_count(3, 3, 15) == 95
