"""Feature hashing on the device (K5, csrc/hash.cu): FNV-1a 32 over
``field 0x1F token`` masked to ``hash_bits`` -- the frozen model contract of
H:1-50, bit-exact.  Batches of (field, token) strings are packed into one
byte buffer + int64 offsets and hashed in one launch.
"""

from __future__ import annotations

import hashlib
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .errors import ContractError

FNV32_OFFSET = 0x811C9DC5  # H:15
FNV32_PRIME = 0x01000193  # H:16
FNV64_OFFSET = 0xCBF29CE484222325  # H:17
FNV64_PRIME = 0x00000100000001B3  # H:18
FIELD_TOKEN_SEP = b"\x1f"  # H:22
MIN_HASH_BITS = 10  # H:24
MAX_HASH_BITS = 29  # H:25


def pack_strings(items) -> tuple[np.ndarray, np.ndarray]:
    """list[bytes] -> (uint8 blob, int64 offsets[n+1])."""
    lens = np.fromiter((len(b) for b in items), dtype=np.int64, count=len(items))
    off = np.zeros(len(items) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    blob = np.frombuffer(b"".join(items), np.uint8) if len(items) else np.zeros(0, np.uint8)
    return blob, off


def hash_bytes(blob, offsets, bits: int = 32, device="cuda") -> torch.Tensor:
    """uint32 FNV-1a of each item, masked to ``bits`` (device tensor, int64 view)."""
    dev = torch.device(device)
    b = torch.as_tensor(np.ascontiguousarray(blob), dtype=torch.uint8).to(dev)
    o = torch.as_tensor(np.ascontiguousarray(offsets), dtype=torch.int64).to(dev)
    n = o.numel() - 1
    out = torch.empty(max(n, 0), dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().fw_hash_fnv1a32(b.data_ptr() if b.numel() else o.data_ptr(),
                                          o.data_ptr(), n, bits, out.data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream),
               "fw_hash_fnv1a32")
    return out.to(torch.int64) & 0xFFFFFFFF


def hash_features(pairs, hash_bits: int, device="cuda") -> torch.Tensor:
    """[(field_name, token)] -> bucket indices (H:42-50) on the device."""
    if not MIN_HASH_BITS <= hash_bits <= MAX_HASH_BITS:
        raise ContractError(
            f"hash_bits must be in [{MIN_HASH_BITS}, {MAX_HASH_BITS}], got {hash_bits}")
    items = [f.encode("utf-8") + FIELD_TOKEN_SEP + t.encode("utf-8") for f, t in pairs]
    blob, off = pack_strings(items)
    return hash_bytes(blob, off, hash_bits, device)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def fnv1a32(data: bytes) -> int:
    """32-bit FNV-1a of a byte string (H:28-32), computed by K5 on the device."""
    blob, off = pack_strings([bytes(data)])
    return int(hash_bytes(blob, off, 32, _device())[0].item())


def fnv1a64(data: bytes) -> int:
    """64-bit FNV-1a (H:35-39): serial by definition, the library's host routine."""
    import ctypes
    buf = bytes(data)
    return int(_lib.lib().fw_fnv1a64_host(ctypes.c_char_p(buf), len(buf)))


@lru_cache(maxsize=1 << 20)
def hash_feature(field_name: str, token: str, hash_bits: int) -> int:
    """Map (field, token) to a stable index below 2**hash_bits (H:42-50), K5 on
    the device; cached like the reference (H:42)."""
    return int(hash_features([(field_name, token)], hash_bits, _device())[0].item())


def content_digest(data) -> int:
    """64-bit digest of a byte buffer keying patches against their base (H:53-59):
    blake2b-64, little-endian, as the reference defines it."""
    return int.from_bytes(hashlib.blake2b(data, digest_size=8).digest(), "little")
