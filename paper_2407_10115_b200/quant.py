"""16-bit weight quantisation on the device (SPEC S:298-385 weight-transfer;
PAPER.md:291-305).  No reference code exists for this module; the semantics
are SPEC's, with the precision choices pinned in SURVEY.md 8(a) row Q and
implemented bit-exactly by K4 (csrc/quant.cu):

    header  w_min = f32(floor_beta(min W)), bucket = f32((ceil_alpha(max W) - that)/65536)
    index   clamp(rint((f64(w) - f64(w_min)) / f64(bucket)), 0, 65535)
    value   w_min + index * bucket   (f32 multiply, then f32 add)

"Per-table" = one header per store block (lr+bias, ffm, each MLP W and b).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import torch

from . import _lib
from .errors import ContractError, FormatError, NumericError

FWQ_MAGIC = b"FWQ1"
FWQ_VERSION = 1
DEFAULT_ALPHA = 4
DEFAULT_BETA = 4


def _stream():
    return torch.cuda.current_stream().cuda_stream


def minmax(w: torch.Tensor):
    """(min, max) of a device f32 tensor; NumericError with the offset of the
    first non-finite weight."""
    if w.dtype != torch.float32 or not w.is_cuda:
        raise ContractError("minmax wants a CUDA f32 tensor")
    w = w.contiguous()
    if w.numel() == 0:
        raise ContractError("quantize of an empty table")
    mm = torch.empty(2, dtype=torch.float32, device=w.device)
    bad = torch.full((1,), -1, dtype=torch.int64, device=w.device)
    _lib.check(_lib.lib().fwq_minmax(w.data_ptr(), w.numel(), mm.data_ptr(), bad.data_ptr(),
                                     _stream()), "fwq_minmax")
    bad_h = int(bad.item()) & ((1 << 64) - 1)
    if bad_h != (1 << 64) - 1:
        raise NumericError(f"non-finite weight at offset {bad_h}", block="quantize")
    lo, hi = mm.tolist()
    return np.float32(lo), np.float32(hi)


def header(wmin, wmax, alpha=DEFAULT_ALPHA, beta=DEFAULT_BETA):
    """(w_min f32, bucket f32) with directional rounding."""
    hmin = ctypes.c_float()
    hb = ctypes.c_float()
    _lib.check(_lib.lib().fwq_header(float(wmin), float(wmax), alpha, beta, ctypes.byref(hmin),
                                     ctypes.byref(hb)), "fwq_header")
    return np.float32(hmin.value), np.float32(hb.value)


def quantize_tensor(w: torch.Tensor, alpha=DEFAULT_ALPHA, beta=DEFAULT_BETA):
    """-> (w_min f32, bucket f32, u16 device tensor of w's shape)."""
    w = w.contiguous()
    lo, hi = minmax(w.view(-1))
    hmin, hb = header(lo, hi, alpha, beta)
    q = torch.empty(w.shape, dtype=torch.uint16, device=w.device)
    _lib.check(_lib.lib().fwq_quantize(w.data_ptr(), w.numel(), float(hmin), float(hb),
                                       q.data_ptr(), _stream()), "fwq_quantize")
    return hmin, hb, q


def dequantize_tensor(q: torch.Tensor, hmin, hb) -> torch.Tensor:
    """w' = w_min + idx*bucket, bit-exact f32."""
    q = q.contiguous()
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    _lib.check(_lib.lib().fwq_dequantize(q.data_ptr(), q.numel(), float(hmin), float(hb),
                                         out.data_ptr(), _stream()), "fwq_dequantize")
    return out


def take_rows(t: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    """t[rows] for any table dtype (torch has no CUDA indexing for uint16)."""
    if t.dtype == torch.uint16:
        return t.view(torch.int16)[rows].view(torch.uint16).contiguous()
    return t[rows].contiguous()


def quantize_store(store, alpha=DEFAULT_ALPHA, beta=DEFAULT_BETA):
    """f32 WeightStore -> serving store with u16 lr/ffm tables (dequantised
    inline by K1/K3) and MLP weights replaced by their dequantised values.

    Returns (store_u16, blobs) where blobs maps table name -> (w_min, bucket,
    u16 tensor) -- the per-table FWQ1 payloads."""
    from .model import WeightStore
    if store.wdtype != "f32":
        raise ContractError("quantize_store wants an f32 store")
    out = WeightStore(store.config, store.device, "u16", with_optimizer=False, _alloc=False)
    blobs = {}
    for name, t in store.blocks(include_optimizer=False):
        hmin, hb, q = quantize_tensor(t, alpha, beta)
        blobs[name] = (hmin, hb, q)
        out.q_headers[name] = (float(hmin), float(hb))
    out.lr = blobs["lr"][2]
    out.ffm = blobs["ffm"][2]
    out.nn_layers = []
    for i in range(len(store.nn_layers)):
        hw, bw, qw = blobs[f"W{i}"]
        hbias, bbias, qb = blobs[f"b{i}"]
        out.nn_layers.append((dequantize_tensor(qw, hw, bw), dequantize_tensor(qb, hbias, bbias)))
    out.version = store.version
    return out, blobs


def to_fwq_blob(hmin, hb, q) -> bytes:
    """FWQ1 file: magic, version u32, w_min f32, bucket f32, count u64, u16 LE."""
    qh = q.detach().cpu().numpy().astype("<u2").reshape(-1) if isinstance(q, torch.Tensor) \
        else np.asarray(q, "<u2").reshape(-1)
    return (FWQ_MAGIC + struct.pack("<Iffq", FWQ_VERSION, float(hmin), float(hb), qh.size)
            + qh.tobytes())


def from_fwq_blob(data: bytes):
    """Parse an FWQ1 blob -> (w_min, bucket, u16 numpy); FormatError if malformed."""
    if len(data) < 24 or data[:4] != FWQ_MAGIC:
        raise FormatError("not a quantized blob (bad magic)")
    ver, hmin, hb, count = struct.unpack("<Iffq", data[4:24])
    if ver != FWQ_VERSION:
        raise FormatError(f"unsupported quantized blob version {ver}")
    if count < 0 or len(data) != 24 + 2 * count:
        raise FormatError("truncated quantized blob")
    return np.float32(hmin), np.float32(hb), np.frombuffer(data[24:], "<u2").copy()
