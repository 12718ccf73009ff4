"""ctypes binding of the in-tree C-ABI library (include/gf_b200.h).

The library is REQUIRED: there is no CPU fallback.  If ``libgf_b200.so`` is
missing, importing the functional API raises with the build command.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgf_b200.so")

GF_F32, GF_F64 = 0, 1
GF_OK, GF_ERR_ARG, GF_ERR_WORKSPACE, GF_ERR_CUDA, GF_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
STATUS_NONFINITE_INPUT, STATUS_NONFINITE_OUTPUT, STATUS_DEGENERATE = 1, 2, 4

_p, _i64, _i, _d, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_size_t

# name -> (restype, argtypes); exactly the symbols declared in include/gf_b200.h
SIGNATURES = {
    "gf_version": (_i, []),
    "gf_last_error": (C.c_char_p, []),
    "gf_sm_count": (_i, []),
    "gf_check_finite": (_i, [_i, _p, _i64, _p, _p]),
    "gf_mean_filter": (_i, [_i, _p, _p, _i64, _i64, _i64, _i, _p]),
    "gf_mean_filter_adjoint": (_i, [_i, _p, _p, _i64, _i64, _i64, _i, _p]),
    "gf_bilinear_resize": (_i, [_i, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gf_bilinear_resize_adjoint": (_i, [_i, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gf_joint_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_joint_fwd": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i, _d, _p,
                          _sz, _p, _p]),
    "gf_joint_bwd": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64,
                          _i, _d, _p, _sz, _p, _p]),
    "gf_joint_bwd_band": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                               _i64, _i, _d, _i64, _p, _sz, _p, _p]),
    "gf_joint_split_threshold": (_i64, []),
    "gf_joint_fwd_mode": (_i, [_i]),
    "gf_joint_coeffs": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _d, _p, _p]),
    "gf_joint_apply": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p]),
    "gf_joint_fwd_tape": (_i, [_i, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i,
                               _d, _p, _sz, _p, _p]),
    "gf_joint_bwd_tape": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64,
                               _i64, _i64, _i, _d, _i64, _p, _sz, _p, _p]),
    "gf_highres_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_highres_fwd": (_i, [_i, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _d, _p, _sz, _p,
                            _p]),
    "gf_highres_bwd": (_i, [_i, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _d, _p,
                            _sz, _p, _p]),
    "gn_param_count": (_i64, [_i64, _i64, _i64]),
    "gn_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i64]),
    "gn_forward": (_i, [_i, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p, _sz, _p, _p]),
    "gn_backward": (_i, [_i, _p, _p, _p, _p, _i, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p,
                         _sz, _p, _p]),
    "gn_backward_reuse": (_i, [_i, _p, _p, _p, _p, _i, _p, _i64, _i64, _i64, _i64, _i64, _i64, _p,
                         _sz, _p, _p]),
    "gn_is_fused": (_i, [_i, _i64, _i64, _i64, _i64, _i64]),
    "gf_mse_loss": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _sz, _p]),
    "gf_mse_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "gf_joint_mse_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_joint_mse_bwd": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                              _i64, _i, _d, _p, _sz, _p, _p]),
    "gnk_param_count": (_i64, [_i64, _i64, _i64, _i]),
    "gnk_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i, _i64, _i64]),
    "gnk_forward": (_i, [_i, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _i, _i64, _i64, _p, _sz, _p,
                         _p]),
    "gnk_backward": (_i, [_i, _p, _p, _p, _p, _i, _p, _i64, _i64, _i64, _i64, _i, _i, _i64, _i64,
                          _p, _sz, _p, _p]),
    "gf_channel_mean": (_i, [_i, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gf_channel_mean_adjoint": (_i, [_i, _p, _p, _i64, _i64, _i64, _i64, _i64, _p]),
    "gf_adam_step": (_i, [_i, _p, _p, _p, _p, _i64, _i, _d, _p, _p]),
    "gf_highres_host_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i]),
    "gf_highres_fwd_host": (_i, [_i, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _d, _p, _sz,
                                 _p]),
    "gf_joint_host_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_joint_fwd_host": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i, _d,
                               _p, _sz, _p]),
    "gf_joint_fwd_bwd_host_workspace_bytes": (_sz, [_i, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_joint_fwd_bwd_host": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64,
                                   _i64, _i64, _i, _d, _p, _sz, _p]),
    "gf_conv2d_fwd": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _i, _p]),
    "gf_conv2d_bwd": (_i, [_i, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _i,
                           _p]),
    "gf_adaptive_norm_workspace_bytes": (_sz, [_i64, _i64]),
    "gf_adaptive_norm_fwd": (_i, [_i, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _sz, _p]),
    "gf_adaptive_norm_bwd": (_i, [_i, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _p,
                                  _sz, _p]),
    "gf_image_unpack_u8": (_i, [_i, _p, _p, _i64, _i64, _i64, _p]),
    "gf_image_pack_u8": (_i, [_i, _p, _p, _i64, _i64, _i64, _p]),
}

# test hooks exported by the library but not part of the public header
EXTRA = {
    "gf_force_generic": (_i, [_i]),
    "gf_highres_variant": (_i, [_i]),
    "gf_joint_bwd_lr_variant": (_i, [_i]),
    "gf_joint_mse_variant": (_i, [_i]),
    "gf_joint_fwd_variant": (_i, [_i]),
    "gf_gn_bwd_variant": (_i, [_i]),
    "gf_joint_bwd_hr_variant": (_i, [_i]),
    "gf_joint_bwd_hr_tile": (_i, [_i]),
    "gf_joint_is_fused": (_i, [_i, _i64, _i64, _i64, _i64, _i64, _i64, _i]),
    "gf_highres_fwd_is_fused": (_i, [_i, _i64, _i64, _i64, _i64, _i64, _i]),
}

_LIB = None


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load and type the library (raises LibraryMissing if it is not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is missing: build it with `python -m paper_1803_05619_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in {**SIGNATURES, **EXTRA}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def last_error() -> str:
    return load().gf_last_error().decode(errors="replace")


class CudaError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if rc == GF_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == GF_ERR_ARG:
        raise ValueError(msg)
    if rc == GF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaError(msg)
