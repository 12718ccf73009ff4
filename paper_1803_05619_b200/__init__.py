"""B200-native guided filtering layer (arXiv 1803.05619), drop-in for the
reference package's layer API (``/root/reference/pkg/src/guidedfilter``).

Public names mirror gf/__init__.py:10-53 for the layer path.  All arithmetic
is done by hand-written sm_100a CUDA kernels in the in-tree ``libgf_b200.so``
(C ABI: include/gf_b200.h); there is no CPU fallback.
"""

from .guided import (
    VARIANT_HIGHRES,
    VARIANT_JOINT,
    DegenerateWindowError,
    GuidedFilterGrads,
    GuidedFilterParams,
    GuidedFilterTape,
    backward,
    forward_highres,
    forward_joint,
)
from .guidance import AdaptiveNorm, ConvLayer, FixedChannelMeanGuidance, GuidanceNet
from .filters import bilinear_resize, bilinear_resize_adjoint, mean_filter, mean_filter_adjoint
from .training import affine_target, joint_mse_backward, mse_loss, train_step
from .nn import FastGuidedFilter, FullResGuidedFilter
from .host import forward_backward_joint_host, forward_highres_host, forward_joint_host
from .upsampler import (TASKS, AdamState, GuidedUpsampler, PipelineTape, TrainConfig,
                        TrainingError, adam_step, build_model, load_checkpoint, make_dataset,
                        save_checkpoint, synthetic_images, train, train_loop)
from . import fileio

__version__ = "0.1.0"

__all__ = [
    "DegenerateWindowError", "GuidedFilterGrads", "GuidedFilterParams", "GuidedFilterTape",
    "VARIANT_HIGHRES", "VARIANT_JOINT", "backward", "forward_highres", "forward_joint",
    "GuidanceNet", "bilinear_resize", "bilinear_resize_adjoint", "mean_filter",
    "mean_filter_adjoint", "affine_target", "mse_loss", "joint_mse_backward", "train_step", "FastGuidedFilter",
    "FullResGuidedFilter", "forward_highres_host", "forward_joint_host",
    "forward_backward_joint_host",
    "FixedChannelMeanGuidance", "AdamState", "GuidedUpsampler", "PipelineTape", "TrainConfig",
    "TrainingError", "adam_step", "build_model", "train", "AdaptiveNorm", "ConvLayer",
    "make_dataset", "synthetic_images", "TASKS", "save_checkpoint", "load_checkpoint",
    "train_loop", "fileio",
]
