"""ctypes binding of ``libdquant_b200.so`` (the C ABI in include/dquant_b200.h).

There is no fallback: if the library is missing or no CUDA device is present,
compute calls raise.  ``torch`` is imported first so the process already holds
the CUDA runtime the library links against; torch is used only for device
memory and streams.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int32, c_int64, c_size_t, c_uint16, c_void_p

import torch

from . import errors

# DQ_LIB: an alternative build of the same library (profiling variants); the in-tree one by default
LIB_PATH = os.environ.get("DQ_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdquant_b200.so")

DQ_OK = 0
DQ_F32, DQ_F16 = 0, 1
LAYOUT_REF, LAYOUT_KTILE, LAYOUT_VTILE = 0, 1, 2
FLAG_NONFINITE, FLAG_RANGE_OVERFLOW, FLAG_JACOBI_NOCONV = 1, 2, 4
I2_PAD = 64

_STATUS = {
    1: errors.UnsupportedBits,
    2: errors.ShapeMismatch,
    3: errors.CorruptPayload,
    4: errors.NonFiniteInput,
    5: errors.RangeOverflow,
    6: ValueError,
    7: errors.CudaFailure,
    8: errors.Unsupported,
}


class Plan2(ctypes.Structure):
    _fields_ = [("i1", c_int64), ("i2", c_int64), ("j1", c_int64), ("j2", c_int64), ("r", c_int64)]


class Segment(ctypes.Structure):
    """dq_segment (include/dquant_b200.h)."""

    _fields_ = [
        ("k_codes", c_void_p),
        ("v_codes", c_void_p),
        ("k_g0", c_void_p),
        ("v_g0", c_void_p),
        ("k_scale", c_float),
        ("v_scale", c_float),
        ("T", c_int32),
        ("i1", c_int32),
        ("i2", c_int32),
        ("r", c_int32),
        ("i2p", c_int32),
        ("unit", c_int32),
        ("token0", c_int32),
        ("pad_", c_int32),
        ("k_ch", c_void_p),
        ("v_ch", c_void_p),
    ]


class AttnArgs(ctypes.Structure):
    """dq_attn_args (include/dquant_b200.h)."""

    _fields_ = [
        ("q", c_void_p),
        ("out", c_void_p),
        ("segs", c_void_p),
        ("nseg", c_int32),
        ("units", c_int32),
        ("g", c_int32),
        ("bits", c_int32),
        ("tail_k", c_void_p),
        ("tail_v", c_void_p),
        ("tail_len", c_void_p),
        ("tail_cap", c_int32),
        ("chunk_b", c_int32),
        ("sm_scale", c_float),
        ("work", c_void_p),
        ("nwork", c_int32),
        ("max_parts", c_int32),
        ("unit_part0", c_void_p),
        ("work_part", c_void_p),
        ("unit_nparts", c_void_p),
        ("sched", c_void_p),
        ("part_o", c_void_p),
        ("part_ml", c_void_p),
        ("phases", c_int32),
        ("nctas", c_int32),
        ("trace", c_void_p),
        ("wimg", c_void_p),
        ("wimg_stride", c_int64),
        ("app_k", c_void_p),
        ("app_v", c_void_p),
        ("head_groups", c_int32),
        ("path", c_int32),
        ("asym", c_int32),
        ("out_bf16", c_int32),
    ]


# name -> (restype, argtypes); every symbol include/dquant_b200.h declares
SIGNATURES = {
    "dq_last_error": (c_char_p, []),
    "dq_version": (c_int32, []),
    "dq_plan_shapes": (c_int32, [c_int64, c_int64, c_int32, POINTER(c_int64), POINTER(c_int64)]),
    "dq_make_plan2": (c_int32, [c_int64, c_int64, POINTER(Plan2)]),
    "dq_layout_bytes": (c_int32, [POINTER(Plan2), c_int32, c_int32, POINTER(c_int64)]),
    "dq_pack": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p]),
    "dq_unpack": (c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p, c_void_p]),
    "dq_quantize_workspace_size": (c_int32, [c_int64, POINTER(c_size_t)]),
    "dq_quantize_rtn": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                  c_void_p]),
    "dq_quantize_rtn_f64": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                      c_void_p]),
    "dq_dequantize": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p]),
    "dq_decompose_workspace_size": (c_int32, [c_int64, c_int64, c_int64, POINTER(c_size_t)]),
    "dq_decompose_batched": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_size_t, c_void_p]),
    "dq_sym_eig_batched": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dq_decompose_plan_batched": (c_int32, [c_void_p, c_int32, c_int64, POINTER(Plan2), c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_size_t, c_void_p]),
    "dq_deco_quantize_batched": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_int64, c_int32, c_int32, c_void_p,
                                           c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "dq_deco_quantize_asym_batched": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_int64, c_int32, c_int32,
                                                c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_size_t,
                                                c_void_p]),
    "dq_core0_relayout": (c_int32, [c_void_p, c_int64, POINTER(Plan2), c_void_p, c_int32, c_void_p, c_void_p]),
    "dq_deco_dequantize_batched": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_int64,
                                             c_int64, c_int32, c_void_p, c_int32, c_void_p]),
    "dq_relayout": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int32, c_int64, c_int64, POINTER(Plan2),
                              c_int32, c_void_p]),
    "dq_fused_matmul_t": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_int64, c_int64,
                                    c_int32, c_void_p, c_void_p, c_void_p]),
    "dq_fused_matmul": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_int64, c_int64,
                                  c_int32, c_void_p, c_void_p, c_void_p]),
    "dq_attention_plan": (c_int32, [POINTER(Segment), c_int32, c_int32, c_int32, c_int32, POINTER(c_int32),
                                    POINTER(c_int32), POINTER(c_int32), POINTER(c_int32), POINTER(c_int32),
                                    POINTER(c_int32)]),
    "dq_attention_ctas": (c_int32, [c_int32, c_int32, POINTER(c_int32)]),
    "dq_decode_attention": (c_int32, [POINTER(AttnArgs), c_void_p]),
    "dq_attention_g0v_dtype": (c_int32, [c_int32, c_int32, c_int32, c_int32, POINTER(c_int32)]),
    "dq_attention_wimg_bytes": (c_int32, [c_int32, POINTER(c_int64)]),
    "dq_tail_append": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "dq_model_add_rmsnorm": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_float,
                                       c_void_p]),
    "dq_model_qkv_rope": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_float, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "dq_model_silu_mul": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
}

_LIB = None


def lib():
    """The loaded library (loaded once).  Raises ImportError when it is not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2405_12591_b200.build` "
                "(there is no CPU fallback)"
            )
        handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("DQ_LIB") and not hasattr(handle, name):
                continue  # an older variant build (A/B measurements): bind what it has
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().dq_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status != DQ_OK:
        cls = _STATUS.get(status, errors.DquantError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise errors.Unsupported("the DecoQuant kernels need a CUDA (sm_100a) device; none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def plan2(rows: int, cols: int) -> Plan2:
    p = Plan2()
    check(lib().dq_make_plan2(rows, cols, ctypes.byref(p)), "plan")
    return p


def layout_bytes(p: Plan2, bits: int, layout: int) -> int:
    out = c_int64()
    check(lib().dq_layout_bytes(ctypes.byref(p), bits, layout, ctypes.byref(out)), "layout_bytes")
    return out.value


def raise_flags(flags, what: str) -> None:
    """Read the device flags word (synchronises) and raise the matching error."""
    f = int(flags.item()) if isinstance(flags, torch.Tensor) else int(flags)
    if f & FLAG_NONFINITE:
        raise errors.NonFiniteSvdInput(f"{what}: input contains NaN or infinity")
    if f & FLAG_RANGE_OVERFLOW:
        raise errors.RangeOverflow(f"{what}: values outside the symmetric range")
    if f & FLAG_JACOBI_NOCONV:
        raise errors.NoConvergence(f"{what}: Jacobi eigensolver did not converge")


__all__ = ["lib", "check", "Plan2", "Segment", "AttnArgs", "SIGNATURES", "c_uint16"]
