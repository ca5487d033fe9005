"""Weight transfer (SPEC module weight-transfer): LEB128 varints and
FWP1 byte patches between two weight files, plus the quantised update
pipeline.  No reference code exists for this module; the SPEC's
examples pin it and `oracle/` restates it for the tests.

The diff and the op encoding run on the GPU (K7, csrc/patch.cu) over device
copies of both files -- a data-parallel pass at HBM speed; applying a patch
parses the op headers on the host (each op's position depends on the one
before, by format) and scatters the payloads on the device.  The FNV-1a 64
digests in the header are serial by definition and are computed on
the host by the library (`fw_fnv1a64_host`).

File format: magic ``FWP1``, version u32, source digest u64, target
digest u64, target length u64 (little-endian), then ``varint(skip)
varint(length) payload`` triples to the end, ``skip`` relative to the end of
the previous op, differing runs closer than ``GAP_MERGE`` = 4 bytes merged.
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import torch

from . import _lib
from .errors import ContractError, CorruptionError, FormatError, StaleBaseError

PATCH_MAGIC = b"FWP1"
PATCH_VERSION = 1
GAP_MERGE = 4
HEADER = struct.Struct("<4sIQQQ")


def encode_varint(n: int) -> bytes:
    """LEB128 base-128 little-endian groups, continuation high bit."""
    if n < 0 or n >= 1 << 64:
        raise ContractError("varint takes an unsigned 64-bit integer")
    out = bytearray()
    while n >= 0x80:
        out.append((n & 0x7F) | 0x80)
        n >>= 7
    out.append(n)
    return bytes(out)


def decode_varint(buf, pos: int = 0):
    """-> (value, bytes consumed); > 10 bytes or truncation -> FormatError."""
    n = 0
    for i in range(10):
        if pos + i >= len(buf):
            raise FormatError("truncated varint")
        b = buf[pos + i]
        n |= (b & 0x7F) << (7 * i)
        if not b & 0x80:
            if n >= 1 << 64:
                raise FormatError("varint overflow")
            return n, i + 1
    raise FormatError("varint longer than 10 bytes")


def digest(data) -> int:
    """FNV-1a 64 over the whole content."""
    a = _host_u8(data)
    return int(_lib.lib().fw_fnv1a64_host(a.ctypes.data, a.size))


def _host_u8(data) -> np.ndarray:
    if isinstance(data, torch.Tensor):
        return data.detach().reshape(-1).view(torch.uint8).cpu().numpy()
    return np.frombuffer(bytes(data) if not isinstance(data, (bytes, bytearray, memoryview))
                         else data, np.uint8)


def _device_u8(data, device) -> torch.Tensor:
    if isinstance(data, torch.Tensor) and data.is_cuda:
        return data.detach().reshape(-1).view(torch.uint8)
    a = _host_u8(data)
    t = torch.empty(a.size, dtype=torch.uint8, device=device)
    if a.size:
        t.copy_(torch.from_numpy(a.copy()))
    return t


def _stream(device):
    return torch.cuda.current_stream(device).cuda_stream


def create_patch(old, new, device="cuda:0") -> bytes:
    """Patch turning ``old`` into ``new``; bytes, numpy or torch inputs."""
    device = torch.device(device)
    lib = _lib.lib()
    od, nd = _device_u8(old, device), _device_u8(new, device)
    n_new = nd.numel()
    scratch = torch.empty(max(int(lib.fwp_scratch_bytes(n_new)), 64), dtype=torch.uint8,
                          device=device)
    s = _stream(device)
    n_ops = ctypes.c_int64(0)
    _lib.check(lib.fwp_diff_count(od.data_ptr(), od.numel(), nd.data_ptr(), n_new,
                                  scratch.data_ptr(), ctypes.byref(n_ops), s), "fwp_diff_count")
    k = n_ops.value
    ops = b""
    if k:
        starts = torch.empty(k, dtype=torch.int64, device=device)
        ends = torch.empty(k, dtype=torch.int64, device=device)
        _lib.check(lib.fwp_diff_ops(od.data_ptr(), od.numel(), nd.data_ptr(), n_new,
                                    scratch.data_ptr(), starts.data_ptr(), ends.data_ptr(), s),
                   "fwp_diff_ops")
        offsets = torch.empty(k, dtype=torch.int64, device=device)
        total = ctypes.c_int64(0)
        _lib.check(lib.fwp_encode_size(starts.data_ptr(), ends.data_ptr(), k, offsets.data_ptr(),
                                       scratch.data_ptr(), ctypes.byref(total), s),
                   "fwp_encode_size")
        out = torch.empty(total.value, dtype=torch.uint8, device=device)
        _lib.check(lib.fwp_encode(nd.data_ptr(), starts.data_ptr(), ends.data_ptr(),
                                  offsets.data_ptr(), k, out.data_ptr(), s), "fwp_encode")
        ops = out.cpu().numpy().tobytes()
    head = HEADER.pack(PATCH_MAGIC, PATCH_VERSION, digest(old), digest(new), n_new)
    return head + ops


def apply_patch(old, patch, device="cuda:0") -> bytes:
    """Apply a patch: StaleBaseError if ``old`` is not the source,
    FormatError for a malformed op stream, CorruptionError if the result's
    digest does not match."""
    device = torch.device(device)
    lib = _lib.lib()
    patch = bytes(patch)
    if len(patch) < HEADER.size:
        raise FormatError("truncated patch header")
    magic, ver, src, dst, tlen = HEADER.unpack_from(patch)
    if magic != PATCH_MAGIC:
        raise FormatError("not a patch (bad magic)")
    if ver != PATCH_VERSION:
        raise FormatError(f"unsupported patch version {ver}")
    if digest(old) != src:
        raise StaleBaseError("patch was made against a different source")
    body = np.frombuffer(patch, np.uint8)[HEADER.size:]
    n_ops = ctypes.c_int64(0)
    _lib.check(lib.fwp_parse_ops(body.ctypes.data, body.size, tlen, None, None, None, 0,
                                 ctypes.byref(n_ops)), "fwp_parse_ops")
    k = n_ops.value
    dst_off = np.empty(k, np.int64)
    src_off = np.empty(k, np.int64)
    lens = np.empty(k, np.int64)
    if k:
        _lib.check(lib.fwp_parse_ops(body.ctypes.data, body.size, tlen, dst_off.ctypes.data,
                                     src_off.ctypes.data, lens.ctypes.data, k,
                                     ctypes.byref(n_ops)), "fwp_parse_ops")
    od = _device_u8(old, device)
    out = torch.zeros(tlen, dtype=torch.uint8, device=device)
    m = min(tlen, od.numel())
    if m:
        out[:m].copy_(od[:m])
    if k:
        s = _stream(device)
        src_t = torch.from_numpy(body.copy()).to(device)
        t = [torch.from_numpy(a).to(device) for a in (dst_off, src_off, lens)]
        _lib.check(lib.fwp_scatter(out.data_ptr(), src_t.data_ptr(), t[0].data_ptr(),
                                   t[1].data_ptr(), t[2].data_ptr(), k, s), "fwp_scatter")
    res = out.cpu().numpy().tobytes()
    if digest(res) != dst:
        raise CorruptionError("patched bytes do not match the target digest")
    return res


def quantized_blob(store, alpha: int = 4, beta: int = 4) -> bytes:
    """The shipped inference artifact: flat weights without the
    optimizer block (M:651 include_optimizer=False), quantised as ONE table
    with one header, as an FWQ1 blob."""
    from .quant import quantize_tensor, to_fwq_blob
    flat = torch.cat([t.reshape(-1).float() for _, t in store.blocks(include_optimizer=False)])
    hmin, hb, q = quantize_tensor(flat, alpha, beta)
    return to_fwq_blob(hmin, hb, q)


def quantized_update_pipeline(old_blob, new_store, alpha: int = 4, beta: int = 4) -> bytes:
    """quantize(new store) then create_patch(previous blob, new blob)."""
    return create_patch(old_blob, quantized_blob(new_store, alpha, beta), new_store.device)
