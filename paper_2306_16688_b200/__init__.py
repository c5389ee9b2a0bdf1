"""B200-native SRL trainer hot path (arXiv 2306.16688): GAE -> advantage normalisation ->
actor-critic MLP forward/backward with the PPO loss fused into the head GEMM -> NCCL gradient
allreduce -> Adam, behind the C ABI of include/srl.h (libsrl.so, sm_100a)."""
from .srl import (  # noqa: F401
    EXPORTS, NetSpec, PPOContext, SrlError, adv_norm, copy_from_device_ptr, debug_gemm, debug_exchange,
    decode_stats, gae, lib, nccl_unique_id,
)
