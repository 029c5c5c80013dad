"""B200-native MoBA attention (FlashMoBA) behind the reference's operator API.

Drop-in for the hot path of the reference package `moba`
(/root/reference/pkg/src/moba/__init__.py:4-43): the same names for the
routing, attention and key-conv operators, backed by hand-written sm_100a
CUDA kernels in libmoba_b200.so (C ABI: include/moba_b200.h). The
reference's SNR model, TNS1 file I/O, CLI and reports are not part of the
accelerated path and are not re-exported here.
"""

from .core import (
    ConfigError,
    FormatError,
    LengthError,
    MobaConfig,
    MobaError,
    OpCounters,
    PlanValidationError,
    RoutingPlan,
    ShapeError,
    resolve_threads,
)
from .router import CentroidMatrix, build_plan, build_varlen, compute_centroids, select_topk
from .attention import AttentionOutput, MobaAttnFunction, moba_attention, moba_attn, moba_backward, moba_forward
from .keyconv import ConvKernel, key_conv_backward, key_conv_forward, random_kernel
from .pipeline import HostPipeline, moba_fwd_bwd_host
from .graphs import MobaGraphedStep
from .tensorio import RunReport, Tensor, tensor_read, tensor_write


def validate_plan(plan, n_tokens: int, cfg: MobaConfig) -> None:
    """validate_plan (src/core.py:254-296), executed on the GPU."""
    from . import _device
    _device.validate(plan, n_tokens, cfg.block_size_B)


__version__ = "0.1.0"
