"""ctypes binding of libdffm.so (include/dffm.h).

This is the reference-facing plugin boundary: plain C types and device
pointers (``torch.Tensor.data_ptr()``), a cudaStream_t, integer status codes.
There is no fallback: if the library is missing the import of any compute
entry point raises, on CPU-only hosts as well as GPU boxes.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_uint8, c_uint16, c_uint32, \
    c_uint64, c_void_p

from . import errors

LIB_PATH = os.environ.get("DFFM_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libdffm.so")
MAX_LAYERS = 5
TRACE_HEAD = 8  # DFFM_TRACE_HEAD

OK, CONTRACT, FORMAT, NUMERIC, SIZING, CUDA = range(6)
BLOCKS = {0: None, 1: "lr", 2: "ffm", 3: "merge", 4: "nn", 5: "logit", 6: "loss"}
W_F32, W_BF16, W_U16Q = 0, 1, 2
STATUS_CLEAR = (1 << 64) - 1


class DffmModel(ctypes.Structure):
    _fields_ = [
        ("n_fields", c_int32), ("k", c_int32), ("hash_bits", c_int32), ("n_layers", c_int32),
        ("dims", c_int32 * (MAX_LAYERS + 1)), ("wdtype", c_int32), ("_pad", c_int32),
        ("lr", c_void_p), ("ffm", c_void_p),
        ("W", c_void_p * MAX_LAYERS), ("b", c_void_p * MAX_LAYERS),
        ("q_lr_min", c_float), ("q_lr_bucket", c_float),
        ("q_ffm_min", c_float), ("q_ffm_bucket", c_float),
    ]


class DffmTrainState(ctypes.Structure):
    _fields_ = [
        ("lr_acc", c_void_p), ("ffm_acc", c_void_p),
        ("W_acc", c_void_p * MAX_LAYERS), ("b_acc", c_void_p * MAX_LAYERS),
        ("lr_ffm", c_double), ("lr_lr", c_double), ("lr_nn", c_double), ("power_t", c_double),
        ("sparse", c_int32), ("_pad", c_int32),
    ]


# name -> (restype, argtypes); every symbol include/dffm.h declares
SIGNATURES = {
    "dffm_abi_version": (c_int32, []),
    "dffm_last_error": (ctypes.c_char_p, []),
    "dffm_build_id": (ctypes.c_char_p, []),
    "dffm_device_sm_count": (c_int32, [c_int32]),
    "dffm_forward": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_int32, c_int64,
                               c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "dffm_set_forward_family": (c_int32, [c_int32]),
    "dffm_set_event_trace": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "dffm_trace_len": (c_int64, [POINTER(DffmModel)]),
    "dffm_forward_trace": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_int32, c_void_p,
                                     c_void_p]),
    "dffm_grad_scratch_len": (c_int64, [POINTER(DffmModel)]),
    "dffm_loss_gradients": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_int32, c_void_p,
                                      c_int32, c_void_p, c_int64, c_void_p, c_void_p]),
    "dffm_ctx_score": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_int32, c_int32,
                                 c_void_p, c_void_p, c_int32, c_int64, c_int32, c_void_p,
                                 c_void_p, c_void_p]),
    "dffm_ctx_cache_bytes": (c_int64, [POINTER(DffmModel), c_int32, c_int32]),
    "dffm_ctx_build": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_int32, c_int32,
                                 c_int64, c_void_p, c_void_p, c_void_p]),
    "dffm_ctx_score_cached": (c_int32, [POINTER(DffmModel), c_void_p, c_void_p, c_void_p, c_int32,
                                        c_int32, c_void_p, c_void_p, c_int32, c_int64, c_int32,
                                        c_void_p, c_void_p, c_void_p]),
    "dffm_ctx_build_count": (c_int64, []),
    "dffm_train_scratch_bytes": (c_int64, [POINTER(DffmModel), c_int32]),
    "dffm_train_sequential": (c_int32, [POINTER(DffmModel), POINTER(DffmTrainState), c_void_p,
                                        c_void_p, c_void_p, c_int32, c_int64, c_void_p,
                                        c_void_p, c_void_p, c_void_p]),
    "dffm_train_hogwild": (c_int32, [POINTER(DffmModel), POINTER(DffmTrainState), c_void_p,
                                     c_void_p, c_void_p, c_int32, c_int64, c_int32, c_void_p,
                                     c_void_p, c_void_p, c_void_p]),
    "dffm_hogwild_max_workers": (c_int32, [POINTER(DffmModel), c_int32]),
    "fwq_minmax": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "fwq_header": (c_int32, [c_float, c_float, c_int32, c_int32, POINTER(c_float),
                             POINTER(c_float)]),
    "fwq_quantize": (c_int32, [c_void_p, c_int64, c_float, c_float, c_void_p, c_void_p]),
    "fwq_dequantize": (c_int32, [c_void_p, c_int64, c_float, c_float, c_void_p, c_void_p]),
    "fw_hash_fnv1a32": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "dffm_unpack_ragged": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                     c_int32, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
                                     c_void_p]),
    "dffm_launch_count": (c_int64, []),
    "dffm_unpack_packed": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                     c_void_p, c_int64, c_int32, c_int32, c_int64, c_int64,
                                     c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fw_parse_scratch_bytes": (c_int64, [c_int64, c_int64]),
    "fw_parse_lines": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                                 c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_void_p]),
    "fw_parse_emit": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p]),
    "fwp_scratch_bytes": (c_int64, [c_int64]),
    "fwp_diff_count": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, POINTER(c_int64),
                                 c_void_p]),
    "fwp_diff_ops": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
    "fwp_encode_size": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                  POINTER(c_int64), c_void_p]),
    "fwp_encode": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fwp_parse_ops": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                                POINTER(c_int64)]),
    "fwp_scatter": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "fw_fnv1a64_host": (c_uint64, [c_void_p, c_int64]),
    "fw_eval_stream": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
                                 c_void_p]),
}

_lib = None


def lib():
    """Load libdffm.so once; raise loudly when it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.DeviceError(
                f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()). "
                "There is no CPU fallback for the DeepFFM hot path.")
        h = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def last_error() -> str:
    msg = lib().dffm_last_error()
    return msg.decode(errors="replace") if msg else ""


_EXC = {CONTRACT: errors.ContractError, FORMAT: errors.FormatError,
        NUMERIC: errors.NumericError, SIZING: errors.SizingError, CUDA: errors.DeviceError}


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    cls = _EXC.get(rc, errors.FieldwiseError)
    raise cls(f"{what}: {last_error()}" if what else last_error())


def raise_status(word: int, what: str = "", base: int = 0) -> None:
    """Decode a device status word (see include/dffm.h) and raise like the reference."""
    word = int(word)
    if word == STATUS_CLEAR:
        return
    example = (word >> 8) + base
    block = BLOCKS.get((word >> 4) & 0xF)
    code = word & 0xF
    if code == NUMERIC:
        raise errors.NumericError(f"{what}non-finite value in {block} block (example {example})",
                                  block=block, example=example)
    if code == CONTRACT:
        exc = errors.ContractError(f"{what}contract violation at example {example}")
        exc.example = example
        raise exc
    raise errors.FieldwiseError(f"{what}device status {word:#x}")


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


__all__ = ["lib", "check", "raise_status", "DffmModel", "DffmTrainState", "SIGNATURES",
           "STATUS_CLEAR", "W_F32", "W_BF16", "W_U16Q", "stream_handle", "c_uint8", "c_uint16",
           "c_uint32", "c_uint64"]
