"""B200-native BurstAttention (arXiv 2403.09347).

Hot path: LAO (tiled flash-style attention, tcgen05/TMEM/TMA kernels for
sm_100a) + GAO (in-kernel online-softmax merge of each ring hop) + the
double-buffered K/V (and dK/dV) ring over NCCL.  Host code is Python/PyTorch;
all compute goes through the C ABI in include/burst_b200.h.
"""

from .api import PassResult, burst_attn_func, run_ring_pass
from .kernels import check_errors
from .lao import local_backward, local_forward
from .errors import (BurstSimError, ConfigError, CudaError, DeadlockError, MaskError,
                     MissingForwardError, NcclError, NonFiniteError, RingDesyncError, ShapeError,
                     UnsupportedError)
from .schedule import HopPlan, plan_hop, shard, shard_map, unshard

__all__ = [
    "burst_attn_func", "run_ring_pass", "local_forward", "local_backward", "PassResult", "check_errors", "plan_hop", "HopPlan", "shard", "unshard",
    "shard_map", "BurstSimError", "ShapeError", "NonFiniteError", "MaskError", "ConfigError",
    "RingDesyncError", "DeadlockError", "MissingForwardError", "CudaError", "NcclError",
    "UnsupportedError",
]
