"""B200-native DecoQuant (arXiv 2405.12591): MPO decomposition + local-tensor quantization
of KV caches, with a fused dequant decode-attention kernel for sm_100a.

Drop-in for the hot path of the reference ``dquant`` package: the names below
mirror ``dquant/__init__.py:10-77`` for the codec, the MPO factorisation, the
DecoQuant protocol and the KV cache.  Compute runs in ``libdquant_b200.so``
(hand-written CUDA, C ABI in include/dquant_b200.h); there is no CPU fallback.
The batched decode hot path is ``DecodeKvCache`` (attention.py).

Also here: the quantisation-error sweeps of the paper's tables on the device path
(``analysis``; its names are re-exported lazily, as in the reference's
``__init__.py:10-20``) and the DQT1 / DQZ1 interchange files (``formats``).  Out of
scope: the dense tensor primitives (``tensor.py``).
"""

from .compress import (
    CompressionReport,
    QuantizedMpo,
    WorkingSetMeter,
    compression_report,
    deco_dequantize,
    deco_quantize,
    fused_matmul,
    fused_matmul_t,
)
from .kvcache import CacheConfig, KvCache, MemoryLedger, simulate_generation
from .mpo import MpoChain, ShapePlan, decompose, plan_shapes, reconstruct, split_large_small
from .quantize import QuantizedTensor, dequantize, pack, quantize_rtn, unpack

_ANALYSIS = ("ErrorRecord", "OutlierStats", "decomposition_comparison", "default_suite", "iqr_stats",
             "length_sweep", "migration_report", "strategy_sweep", "synth_activations")

__all__ = [
    *_ANALYSIS,
    "CacheConfig",
    "CompressionReport",
    "DecodeKvCache",
    "KvCache",
    "MemoryLedger",
    "MpoChain",
    "QuantizedMpo",
    "QuantizedTensor",
    "ShapePlan",
    "WorkingSetMeter",
    "compression_report",
    "deco_dequantize",
    "deco_quantize",
    "decompose",
    "dequantize",
    "fused_matmul",
    "fused_matmul_t",
    "pack",
    "plan_shapes",
    "quantize_rtn",
    "reconstruct",
    "simulate_generation",
    "split_large_small",
    "unpack",
]

__version__ = "0.1.0"


def __getattr__(name):
    if name == "DecodeKvCache":
        from .attention import DecodeKvCache

        return DecodeKvCache
    if name in _ANALYSIS:  # analysis imports the sweeps' device paths: loaded on first use
        from . import analysis

        return getattr(analysis, name)
    raise AttributeError(name)
