"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side harness.

This module holds NO arithmetic of the method (no GAE, no normalisation, no network, no
loss): only workload shapes (BASELINE.json ``configs``) and a counter-based random
generator that builds trajectory batches with the structure SURVEY.md §8(d) D-1 lays out.
Both sides receive the same arrays from here; neither side's compute lives here.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .gen import (  # noqa: F401
    splitmix64, uniform, normal, make_batch, make_params, shard_columns,
    logp_old_uniform_policy,
)
from .torch_gen import make_batch_device  # noqa: F401
