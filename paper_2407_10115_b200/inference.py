"""Serving with context caching (SPEC inference-engine).

No reference code exists for this module; the contract is
SPEC's: cached scoring equals ``forward`` + ``predict_proba`` on the merged
context+candidate example, the cache is a pure function of (context,
weights version) and a version bump makes it stale.

On the GPU the cache itself (context lr partial, context latent sums
S[x][g][:], ctx x ctx pair values) is built per request inside K3's shared
memory (csrc/ctx.cu) and reused by every candidate of that request; it never
round-trips through HBM.  The host-side ``ContextCache`` records the packed
context, its digest and the store version it is valid for.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractError, StaleCacheError
from .model import WeightStore, _as_device, _status


@dataclass
class ContextCache:
    ctx_idx: torch.Tensor  # [1, Fc, Mc] int32, device
    ctx_val: torch.Tensor  # [1, Fc, Mc] f32, device
    n_ctx_fields: int
    digest: int
    store_version: int


def _digest(idx: np.ndarray, val: np.ndarray) -> int:
    """64-bit digest of sorted (field, index, value-bits) triples."""
    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(idx, np.int32).tobytes())
    h.update(np.ascontiguousarray(val, np.float32).tobytes())
    return int.from_bytes(h.digest(), "little")


def build_context_cache(ctx_idx, ctx_val, store: WeightStore) -> ContextCache:
    """Context fields occupy field ids [0, Fc) (disjoint from the
    candidates').  ``ctx_idx``/``ctx_val``: [Fc, Mc] or [1, Fc, Mc]."""
    ci = np.asarray(ctx_idx.cpu() if isinstance(ctx_idx, torch.Tensor) else ctx_idx)
    cv = np.asarray(ctx_val.cpu() if isinstance(ctx_val, torch.Tensor) else ctx_val)
    if ci.ndim == 2:
        ci, cv = ci[None], cv[None]
    if ci.shape[1] > store.config.n_fields:
        raise ContractError("more context fields than the model has")
    dev = store.device
    return ContextCache(_as_device(ci, torch.int32, dev), _as_device(cv, torch.float32, dev),
                        ci.shape[1], _digest(ci, cv), store.version)


def score_requests(ctx_idx, ctx_val, cand_idx, cand_val, store: WeightStore,
                   out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """Batched K3: ctx [R, Fc, Mc], cand [R, C, F-Fc, Md] -> prob [R, C] (device f32)."""
    dev = store.device
    ci = _as_device(ctx_idx, torch.int32, dev)
    cv = _as_device(ctx_val, torch.float32, dev)
    di = _as_device(cand_idx, torch.int32, dev)
    dv = _as_device(cand_val, torch.float32, dev)
    R, Fc, Mc = ci.shape
    if di.dim() != 4 or di.shape[0] != R or di.shape[2] != store.config.n_fields - Fc:
        raise ContractError(f"candidate layout {tuple(di.shape)} does not match "
                            f"[{R}, C, {store.config.n_fields - Fc}, M]")
    C, Md = di.shape[1], di.shape[3]
    if out is None:
        out = torch.empty((R, C), dtype=torch.float32, device=dev)
    st = _status(dev)
    s = torch.cuda.current_stream(dev)
    st.clear()
    rc = _lib.lib().dffm_ctx_score(store.c_model_ref(), ci.data_ptr(), cv.data_ptr(), Fc, Mc,
                                   di.data_ptr(), dv.data_ptr(), Md, R, C, out.data_ptr(),
                                   st.ptr(), s.cuda_stream)
    _lib.check(rc, "dffm_ctx_score")
    if check:
        st.fetch_async()
        s.synchronize()
        st.raise_if_set("context scorer: ")
    return out


def predict_batch(cache: ContextCache, cand_idx, cand_val, store: WeightStore) -> torch.Tensor:
    """Score the candidates of one request against a cache."""
    if cache.store_version != store.version:
        raise StaleCacheError("context cache built against an older weights version")
    di = _as_device(cand_idx, torch.int32, store.device)
    dv = _as_device(cand_val, torch.float32, store.device)
    if di.dim() == 3:
        di, dv = di[None], dv[None]
    return score_requests(cache.ctx_idx, cache.ctx_val, di, dv, store)[0]
