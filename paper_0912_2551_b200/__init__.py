"""paper_0912_2551_b200 -- B200-native hot path of the statistical model checker
of arXiv:0912.2551 (SSA trajectories verified on the fly against BLTLc
formulas, Wilson-interval stopping rule), behind the C ABI of include/smc.h.

This module is the thin Python binding: argument marshalling only.  Every step
of the path runs in libsmc.so (host C++ + sm_100a CUDA kernels); PyTorch is
used for device memory, streams and torch.distributed process groups.  There
is no CPU fallback: without libsmc.so (or without an sm_100 GPU for the
kernel calls) every call raises.
"""
from ._native import (  # noqa: F401
    SmcError, lib, smc_last_error,
    smc_normal_quantile, smc_wilson_interval, smc_wilson_sample_size, smc_shard_range, smc_window_ring_plan,
    smc_philox_blocks, smc_draw_blocks, smc_set_shard, smc_set_stream,
)
from .api import (  # noqa: F401
    Model, Property, estimate, estimate_with_runner, use_torch, set_allreduce_torch, clear_allreduce,
    COUNTS_KEYS,
)
