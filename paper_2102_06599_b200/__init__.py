"""paper_2102_06599_b200 -- B200-native hot path of arXiv 2102.06599.

Conv-nest execution and the Fisher Potential legality check of the reference
library ``nestopt``, rebuilt as sm_100a CUDA kernels behind a C ABI
(include/nb200.h, libnb200.so).  ``api`` mirrors the reference's operator
API; ``abi`` is the raw ctypes binding.
"""
from .api import (  # noqa: F401
    Batch, ChannelSplit, ConfigError, Context, ConvSpec, CudaError, Error, EvalStats,
    RECHECK_BAND, TIE_BAND, TOLERANCE, TOLERANCE_DEEP, FisherReport, ForwardCache, InvalidSpec, Layer, Network, NoDevice, Precision, Session,
    ShapeMismatch, Unsupported, activation_gradients, conv_dgrad, count_macs,
    default_context, device_count, fp32_split, evaluate, fisher_accepts, fisher_flops, fisher_potential,
    fisher_sharded, shard_batch,
    forward, layer_forward, legality_fisher, make_batch, network_macs, reference_conv,
    repair_network, schedule_lpt,
)
