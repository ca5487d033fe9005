"""Seeded synthetic inputs and weights for the BASELINE workloads.

Everything is generated with torch on the device it will be used on (CPU for
the unit tests, ``cuda:N`` for the bench), so a 2^24-bucket table or a
1M-example batch never round-trips through host numpy.  The recipe:

* ranks r in [1, 2^b] drawn by inverse-CDF search over the truncated Zipf(alpha)
  CDF (``searchsorted(cdf, U, right)+1``) or uniformly;
* rank -> bucket with the reference's own feature hash,
  ``hash_feature(f"f{field}", f"t{r}", b)`` = FNV-1a-32 over
  ``field 0x1F token`` masked to b bits (H:28-50), computed vectorised here
  (bit-exact; checked against the reference in tests/test_synth.py).  The
  "unsalted" variant maps bucket = r-1 in every field (duplicate stress);
* canonical per (example, field): sorted unique indices, duplicate values
  summed (Fe:166-172, Fe:219), padded with sentinel -1 to M slots;
* numeric fields carry LogNormal(0,1) values rounded to f32; categorical 1.0.
"""

from __future__ import annotations

import torch

from .configs import Workload

FNV32_OFFSET = 0x811C9DC5
FNV32_PRIME = 0x01000193
_MASK32 = 0xFFFFFFFF


def _fnv_update(h: int, data: bytes) -> int:
    for b in data:
        h = ((h ^ b) * FNV32_PRIME) & _MASK32
    return h


def hash_ranks(field_ids: torch.Tensor, ranks: torch.Tensor, hash_bits: int) -> torch.Tensor:
    """Bucket of token ``t{r}`` in field ``f{field}`` (int64 tensor, same shape).

    The FNV state after the constant prefix ``f{field} 0x1F t`` is computed
    once per field on the host; the decimal digits of r are then folded in
    vectorised."""
    field_ids = field_ids.to(torch.int64)
    ranks = ranks.to(torch.int64)
    n_f = int(field_ids.max().item()) + 1 if field_ids.numel() else 1
    prefix = torch.tensor([_fnv_update(FNV32_OFFSET, f"f{f}".encode() + b"\x1ft")
                           for f in range(n_f)], dtype=torch.int64, device=ranks.device)
    h = prefix[field_ids]
    nd = torch.ones_like(ranks)
    for p in range(1, 19):
        nd = nd + (ranks >= 10 ** p).to(torch.int64)
    maxd = int(nd.max().item()) if ranks.numel() else 1
    for pos in range(maxd):
        live = nd > pos
        shift = (nd - 1 - pos).clamp(min=0)
        pw = torch.pow(torch.full_like(shift, 10), shift)
        digit = (ranks // pw) % 10
        nh = ((h ^ (digit + 0x30)) * FNV32_PRIME) & _MASK32
        h = torch.where(live, nh, h)
    return h & ((1 << hash_bits) - 1)


def zipf_cdf(n: int, alpha: float, device) -> torch.Tensor:
    # always summed on the host: a device cumsum is a parallel scan whose f64 rounding
    # varies from process to process (a handful of the 10^8 ranks of a cfg5 batch
    # moved between runs), and the seeded inputs are meant to be reproducible
    r = torch.arange(1, n + 1, dtype=torch.float64)
    w = r.pow(-alpha)
    c = torch.cumsum(w, 0)
    return (c / c[-1]).to(device)


def sample_ranks(shape, n: int, dist: str, alpha: float, gen: torch.Generator, device,
                 cdf=None) -> torch.Tensor:
    if dist == "uniform":
        return torch.randint(1, n + 1, shape, generator=gen, device=device, dtype=torch.int64)
    if cdf is None:
        cdf = zipf_cdf(n, alpha, device)
    u = torch.rand(shape, generator=gen, device=device, dtype=torch.float64)
    r = torch.searchsorted(cdf, u.reshape(-1), right=True).reshape(shape) + 1
    return r.clamp_(max=n)


def canonicalize(idx: torch.Tensor, val: torch.Tensor):
    """Sort each [.., M] slot group, merge duplicates (values summed in f64,
    rounded to f32), compact, pad with -1 (Fe:166-172, Fe:219)."""
    big = torch.iinfo(torch.int64).max
    key = torch.where(idx < 0, torch.full_like(idx, big), idx.to(torch.int64))
    key, perm = torch.sort(key, dim=-1, stable=True)
    v = torch.gather(val.to(torch.float64), -1, perm)
    M = idx.shape[-1]
    for j in range(M - 1, 0, -1):
        dup = (key[..., j] == key[..., j - 1]) & (key[..., j] != big)
        v[..., j - 1] = torch.where(dup, v[..., j - 1] + v[..., j], v[..., j - 1])
        key[..., j] = torch.where(dup, torch.full_like(key[..., j], big), key[..., j])
    key, perm = torch.sort(key, dim=-1, stable=True)
    v = torch.gather(v, -1, perm)
    out_idx = torch.where(key == big, torch.full_like(key, -1), key).to(torch.int32)
    out_val = torch.where(key == big, torch.zeros_like(v), v).to(torch.float32)
    return out_idx.contiguous(), out_val.contiguous()


def make_examples(wl: Workload, n: int, seed: int | None = None, device="cpu",
                  hash_bits: int | None = None, salted: bool = True,
                  field_offset: int = 0, n_fields: int | None = None, cdf=None):
    """Padded canonical examples: (idx int32 [n,F,M], val f32 [n,F,M])."""
    device = torch.device(device)
    bits = wl.hash_bits if hash_bits is None else hash_bits
    F = wl.n_fields if n_fields is None else n_fields
    M = wl.max_per_field
    gen = torch.Generator(device=device)
    gen.manual_seed(wl.data_seed if seed is None else seed)
    nb = 1 << bits
    if M > 1:
        counts = torch.randint(1, M + 1, (n, F), generator=gen, device=device)
    else:
        counts = torch.ones((n, F), dtype=torch.int64, device=device)
    ranks = sample_ranks((n, F, M), nb, wl.dist, wl.zipf_alpha, gen, device, cdf)
    fids = (torch.arange(F, device=device) + field_offset).view(1, F, 1).expand(n, F, M)
    if salted:
        buckets = hash_ranks(fids, ranks, bits)
    else:
        buckets = ranks - 1
    val = torch.ones((n, F, M), dtype=torch.float64, device=device)
    for f in wl.numeric_fields:
        if field_offset <= f < field_offset + F:
            z = torch.randn((n, M), generator=gen, device=device, dtype=torch.float64)
            val[:, f - field_offset, :] = torch.exp(z).to(torch.float32).to(torch.float64)
    slot = torch.arange(M, device=device).view(1, 1, M)
    live = slot < counts.unsqueeze(-1)
    buckets = torch.where(live, buckets, torch.full_like(buckets, -1))
    return canonicalize(buckets, val)


def make_labels(n: int, p: float, seed: int, device="cpu") -> torch.Tensor:
    gen = torch.Generator(device=torch.device(device))
    gen.manual_seed(seed)
    return (torch.rand(n, generator=gen, device=device) < p).to(torch.uint8)


def normal_table(numel: int, scale: float, gen: torch.Generator, device,
                 chunk: int = 1 << 28) -> torch.Tensor:
    """N(0, scale) f32 values drawn chunk by chunk in flat order."""
    out = torch.empty(numel, dtype=torch.float32, device=device)
    for c0 in range(0, numel, chunk):
        c1 = min(numel, c0 + chunk)
        out[c0:c1] = torch.randn(c1 - c0, generator=gen, device=device,
                                 dtype=torch.float32) * scale
    return out


def count_features(idx: torch.Tensor) -> int:
    return int((idx >= 0).sum().item())


__all__ = ["hash_ranks", "zipf_cdf", "sample_ranks", "canonicalize", "make_examples",
           "make_labels", "normal_table", "count_features"]
