"""B200-native SLQ hot path of HessFormer (arxiv 2505.11564).

The reference-facing API (specden names, SPEC.md semantics) lives in
``core``; the GPT Hessian-vector-product engine in ``gpt``. Importing the
package loads libspecden_b200.so and fails loudly if it is missing: there is
no CPU fallback.
"""
from ._lib import lib as _load

_load()

from .core import *  # noqa: E402,F401,F403
from .core import (F32, F64, GAUSSIAN, ONE_HOT, RADEMACHER, REDUCE_ORDERED, REDUCE_TREE, REORTH_FULL, REORTH_NONE,  # noqa: E402,F401,E501
                   REORTH_SELECTIVE,
                   Lanczos,
                   LanczosConfig, LanczosResult, OperatorHandle, ProbeSpec, RitzSpectrum, ShardedVector, ShardLayout,
                   WorkerPool)

from . import column_probe, diagnostics, gemm, gpt, mlp, slq  # noqa: E402,F401
