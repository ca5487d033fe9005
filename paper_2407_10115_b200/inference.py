"""Serving with context caching (SPEC inference-engine).

No reference code exists for this module; the contract is
SPEC's: cached scoring equals ``forward`` + ``predict_proba`` on the merged
context+candidate example within 1e-6, the cache is a pure function of
(context, weights version), a version bump makes it stale, and
caches are keyed by a 64-bit digest of the sorted (field_id, feature_index,
value-bits) triples so that a repeated context is built once.

``build_context_cache`` runs K3's build pass (``dffm_ctx_build``) once: the
context lr partial, the context latent sums S[x][g][:] and the ctx x ctx pair
outputs with their moments stay resident in HBM as one blob per request.
``predict_batch(cache, ...)`` scores candidates against that blob
(``dffm_ctx_score_cached``: no context pass); ``ContextCacheMap`` is the
digest-keyed store that reuses a cache across requests until the weights move.
"""

from __future__ import annotations

import hashlib
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractError, StaleCacheError
from .model import StatusWord, WeightStore, _as_device, _status


@dataclass
class ContextCache:
    ctx_idx: torch.Tensor  # [1, Fc, Mc] int32, device
    ctx_val: torch.Tensor  # [1, Fc, Mc] f32, device
    n_ctx_fields: int
    digest: int
    store_version: int
    blob: torch.Tensor | None = None  # device uint8 [cache_bytes]: the built cache


def _digest(idx: np.ndarray, val: np.ndarray) -> int:
    """64-bit digest of the sorted (field_id, feature_index, value-bits) triples
    of a context: independent of slot order and padding."""
    idx = np.asarray(idx).reshape(idx.shape[-2], -1)
    val = np.asarray(val, np.float32).reshape(idx.shape)
    f, m = np.nonzero(idx >= 0)
    trip = np.stack([f.astype(np.int64), idx[f, m].astype(np.int64),
                     val[f, m].view(np.uint32).astype(np.int64)], axis=1)
    trip = trip[np.lexsort((trip[:, 2], trip[:, 1], trip[:, 0]))]
    h = hashlib.blake2b(np.ascontiguousarray(trip).tobytes(), digest_size=8)
    return int.from_bytes(h.digest(), "little")


def build_context_cache(ctx_idx, ctx_val, store: WeightStore) -> ContextCache:
    """Context fields occupy field ids [0, Fc) (disjoint from the
    candidates').  ``ctx_idx``/``ctx_val``: [Fc, Mc] or [1, Fc, Mc].  Runs the
    context pass once on the device (cost independent of the candidates)."""
    ci = np.asarray(ctx_idx.cpu() if isinstance(ctx_idx, torch.Tensor) else ctx_idx)
    cv = np.asarray(ctx_val.cpu() if isinstance(ctx_val, torch.Tensor) else ctx_val)
    if ci.ndim == 2:
        ci, cv = ci[None], cv[None]
    Fc, Mc = ci.shape[1], ci.shape[2]
    if Fc >= store.config.n_fields or Fc < 1:
        raise ContractError("context fields must be a non-empty proper prefix of the model's")
    dev = store.device
    di, dv = _as_device(ci, torch.int32, dev), _as_device(cv, torch.float32, dev)
    lib = _lib.lib()
    cm = store.c_model_ref()
    nbytes = int(lib.dffm_ctx_cache_bytes(cm, Fc, Mc))
    if nbytes < 0:
        _lib.check(_lib.CONTRACT, "dffm_ctx_cache_bytes")
    blob = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    st = _status(dev)
    s = torch.cuda.current_stream(dev)
    st.clear()
    _lib.check(lib.dffm_ctx_build(cm, di.data_ptr(), dv.data_ptr(), Fc, Mc, 1, blob.data_ptr(),
                                  st.ptr(), s.cuda_stream), "dffm_ctx_build")
    st.fetch_async()
    s.synchronize()
    st.raise_if_set("context cache: ")
    return ContextCache(di, dv, Fc, _digest(ci[0], cv[0]), store.version, blob)


class ContextCacheMap:
    """Digest-keyed context caches ("dedupe"): a repeated context reuses
    its device-resident cache; a weights-version bump drops every entry."""

    def __init__(self, store: WeightStore, capacity: int = 4096):
        self.store, self.capacity = store, int(capacity)
        self._map: OrderedDict = OrderedDict()
        self._version = store.version
        self.hits = self.misses = 0

    def get(self, ctx_idx, ctx_val) -> ContextCache:
        if self.store.version != self._version:
            self._map.clear()
            self._version = self.store.version
        ci = np.asarray(ctx_idx.cpu() if isinstance(ctx_idx, torch.Tensor) else ctx_idx)
        cv = np.asarray(ctx_val.cpu() if isinstance(ctx_val, torch.Tensor) else ctx_val)
        key = (ci.shape[-2], _digest(ci.reshape(ci.shape[-2], -1), cv.reshape(ci.shape[-2], -1)))
        hit = self._map.get(key)
        if hit is not None:
            self._map.move_to_end(key)
            self.hits += 1
            return hit
        self.misses += 1
        cache = build_context_cache(ci, cv, self.store)
        self._map[key] = cache
        if len(self._map) > self.capacity:
            self._map.popitem(last=False)
        return cache


def score_requests(ctx_idx, ctx_val, cand_idx, cand_val, store: WeightStore,
                   out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """Batched K3: ctx [R, Fc, Mc], cand [R, C, F-Fc, Md] -> prob [R, C] (device f32);
    each request's context pass runs once inside the kernel."""
    return _score(None, ctx_idx, ctx_val, cand_idx, cand_val, store, out, check)


class HostRequestScorer:
    """Host-buffer entry point of K3: pinned host requests in, host probabilities out.

    The requests are cut into chunks (multiples of the SM count, so every CTA of the
    ring kernel gets the same number of requests); chunk j+1's contexts and
    candidates cross PCIe on the copy stream while K3 scores chunk j on the compute
    stream and chunk j-1's probabilities return on a third stream (two device
    staging buffers in flight).  ``bench.py --workload cfg4`` reports its ``e2e``
    through this call."""

    def __init__(self, store: WeightStore, n_ctx_fields: int, ctx_m: int, n_cand: int,
                 cand_m: int, chunk_requests: int = 296):
        self.store = store
        dev = store.device
        Fd = store.config.n_fields - n_ctx_fields
        if n_ctx_fields < 1 or Fd < 1:
            raise ContractError("context fields must be a non-empty proper prefix of the model's")
        self.shape = (n_ctx_fields, ctx_m, n_cand, Fd, cand_m)
        self.chunk = max(1, int(chunk_requests))
        q = self.chunk
        self.ci = [torch.empty((q, n_ctx_fields, ctx_m), dtype=torch.int32, device=dev) for _ in range(2)]
        self.cv = [torch.empty((q, n_ctx_fields, ctx_m), dtype=torch.float32, device=dev) for _ in range(2)]
        self.di = [torch.empty((q, n_cand, Fd, cand_m), dtype=torch.int32, device=dev) for _ in range(2)]
        self.dv = [torch.empty((q, n_cand, Fd, cand_m), dtype=torch.float32, device=dev) for _ in range(2)]
        self.prob = [torch.empty((q, n_cand), dtype=torch.float32, device=dev) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(dev)
        self.compute_stream = torch.cuda.Stream(dev)
        self.out_stream = torch.cuda.Stream(dev)
        self.status = StatusWord(dev)

    def __call__(self, ctx_idx: torch.Tensor, ctx_val: torch.Tensor, cand_idx: torch.Tensor,
                 cand_val: torch.Tensor, out_host: torch.Tensor, check: bool = True) -> torch.Tensor:
        Fc, Mc, C, Fd, Md = self.shape
        R = int(ctx_idx.shape[0])
        if tuple(ctx_idx.shape) != (R, Fc, Mc) or tuple(cand_idx.shape) != (R, C, Fd, Md):
            raise ContractError(f"request layout {tuple(ctx_idx.shape)} / {tuple(cand_idx.shape)} does "
                                f"not match [R, {Fc}, {Mc}] / [R, {C}, {Fd}, {Md}]")
        lib = _lib.lib()
        cm = self.store.c_model_ref()
        cs, ks, os_ = self.copy_stream, self.compute_stream, self.out_stream
        ks.wait_stream(torch.cuda.current_stream(self.store.device))
        with torch.cuda.stream(ks):
            self.status.clear()
        cs.wait_stream(ks)
        h2d = [torch.cuda.Event(), torch.cuda.Event()]
        scored = [torch.cuda.Event(), torch.cuda.Event()]
        drained = [torch.cuda.Event(), torch.cuda.Event()]
        # a short first chunk, so the first (unoverlapped) copy is short
        bounds, r0 = [], 0
        first = max(1, self.chunk // 2)
        while r0 < R:
            r1 = min(R, r0 + (first if not bounds else self.chunk))
            bounds.append((r0, r1))
            r0 = r1
        for j, (r0, r1) in enumerate(bounds):
            b, n = j & 1, r1 - r0
            with torch.cuda.stream(cs):
                if j >= 2:
                    cs.wait_event(scored[b])  # the staging buffers of chunk j-2 are free
                self.ci[b][:n].copy_(ctx_idx[r0:r1], non_blocking=True)
                self.cv[b][:n].copy_(ctx_val[r0:r1], non_blocking=True)
                self.di[b][:n].copy_(cand_idx[r0:r1], non_blocking=True)
                self.dv[b][:n].copy_(cand_val[r0:r1], non_blocking=True)
                h2d[b].record(cs)
            with torch.cuda.stream(ks):
                ks.wait_event(h2d[b])
                if j >= 2:
                    ks.wait_event(drained[b])  # prob[b] of chunk j-2 has left
                rc = lib.dffm_ctx_score(cm, self.ci[b].data_ptr(), self.cv[b].data_ptr(), Fc, Mc,
                                        self.di[b].data_ptr(), self.dv[b].data_ptr(), Md, n, C,
                                        self.prob[b].data_ptr(), self.status.ptr(), ks.cuda_stream)
                _lib.check(rc, "dffm_ctx_score")
                scored[b].record(ks)
            with torch.cuda.stream(os_):
                os_.wait_event(scored[b])
                out_host[r0:r1].copy_(self.prob[b][:n], non_blocking=True)
                drained[b].record(os_)
        ks.wait_stream(os_)
        with torch.cuda.stream(ks):
            self.status.fetch_async()
        ks.synchronize()
        if check and int(self.status.host.item()) != -1:
            # the status word holds chunk-local candidate numbers: find the first
            # failing chunk again, serially, and report the stream-global candidate
            for r0, r1 in bounds:
                _score(None, ctx_idx[r0:r1], ctx_val[r0:r1], cand_idx[r0:r1], cand_val[r0:r1],
                       self.store, None, True, base=r0 * C)
            self.status.raise_if_set("context scorer: ")
        return out_host


def _score(blob, ctx_idx, ctx_val, cand_idx, cand_val, store, out, check, base=0):
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
    lib = _lib.lib()
    if blob is None:
        rc = lib.dffm_ctx_score(store.c_model_ref(), ci.data_ptr(), cv.data_ptr(), Fc, Mc,
                                di.data_ptr(), dv.data_ptr(), Md, R, C, out.data_ptr(), st.ptr(),
                                s.cuda_stream)
    else:
        rc = lib.dffm_ctx_score_cached(store.c_model_ref(), blob.data_ptr(), ci.data_ptr(),
                                       cv.data_ptr(), Fc, Mc, di.data_ptr(), dv.data_ptr(), Md,
                                       R, C, out.data_ptr(), st.ptr(), s.cuda_stream)
    _lib.check(rc, "dffm_ctx_score")
    if check:
        st.fetch_async()
        s.synchronize()
        st.raise_if_set("context scorer: ", base)
    return out


def predict_batch(cache: ContextCache, cand_idx, cand_val, store: WeightStore) -> torch.Tensor:
    """Score the candidates of one request against a built cache:
    candidate x candidate and candidate x context pairs fresh, the context
    part from the cache."""
    if cache.store_version != store.version:
        raise StaleCacheError("context cache built against an older weights version")
    di = _as_device(cand_idx, torch.int32, store.device)
    dv = _as_device(cand_val, torch.float32, store.device)
    if di.dim() == 3:
        di, dv = di[None], dv[None]
    return _score(cache.blob, cache.ctx_idx, cache.ctx_val, di, dv, store, None, True)[0]
