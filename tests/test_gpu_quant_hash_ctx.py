"""K4 quantisation (bit-exact), K5 hashing (bit-exact) and K3 context cache
(1e-6 absolute) on the GPU."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200 import configs, hashing, inference, quant, synth
from paper_2407_10115_b200.errors import ContractError, NumericError, StaleCacheError
from paper_2407_10115_b200.model import ModelConfig, WeightStore, predict_batch
from tests.golden_io import fixture_flat, load
from tests.remap import compact_oracle

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


# ------------------------------------------------------------------ K4


@pytest.mark.parametrize("n,scale", [(1, 0.1), (3, 1.0), (1001, 0.05), (1 << 20, 0.05),
                                     ((1 << 22) + 3, 2.5)])
def test_quantize_bit_exact(n, scale):
    rng = np.random.default_rng(n)
    w = (rng.standard_normal(n) * scale).astype(np.float32)
    hmin, hb, q = quant.quantize_tensor(torch.from_numpy(w).to(DEV))
    rmin, rb, rq = fo.quantize(w)
    assert (hmin, hb) == (rmin, rb)
    assert np.array_equal(q.cpu().numpy(), rq)
    back = quant.dequantize_tensor(q, hmin, hb).cpu().numpy()
    assert back.tobytes() == fo.dequantize(rmin, rb, rq).tobytes()


def test_quantize_kats_and_errors():
    hmin, hb, q = quant.quantize_tensor(torch.tensor([0.0, 1.0, 0.5], device=DEV))
    assert hmin == 0.0 and hb == np.float32(1 / 65536) and q.cpu().tolist() == [0, 65535, 32768]
    hmin, hb, q = quant.quantize_tensor(torch.full((7,), 0.25, device=DEV))
    assert hb == 0 and (q == 0).all()
    with pytest.raises(ContractError):
        quant.quantize_tensor(torch.zeros(0, device=DEV))
    w = torch.randn(1000, device=DEV)
    w[417] = float("inf")
    w[900] = float("nan")
    with pytest.raises(NumericError, match="offset 417"):
        quant.quantize_tensor(w)


def test_fwq_blob_roundtrip():
    w = torch.randn(12345, device=DEV) * 0.05
    hmin, hb, q = quant.quantize_tensor(w)
    blob = quant.to_fwq_blob(hmin, hb, q)
    assert len(blob) == 24 + 2 * 12345  # S:379; ~half of 4-byte weights
    h2, b2, q2 = quant.from_fwq_blob(blob)
    assert (h2, b2) == (hmin, hb) and np.array_equal(q2, q.cpu().numpy())
    with pytest.raises(Exception):
        quant.from_fwq_blob(blob[:-2])


def test_quantize_store_full_cfg4_table_properties():
    """cfg4-size ffm table (2^24 x 24 x 8): size-independent properties --
    dequantise(quantise(W)) within bucket/2 (+f32 slack), monotone, and an
    exact oracle check on a slice."""
    n = (1 << 24) * 24 * 8
    gen = torch.Generator(device=DEV).manual_seed(1004)
    w = synth.normal_table(n, 0.05, gen, DEV)
    hmin, hb, q = quant.quantize_tensor(w)
    back = quant.dequantize_tensor(q, hmin, hb)
    err = (back.double() - w.double()).abs()
    inner = (q.to(torch.int32) > 0) & (q.to(torch.int32) < 65535)
    slack = 65536 * float(np.spacing(hb)) + 2 * float(np.spacing(np.float32(w.abs().max().item())))
    assert err[inner].max().item() <= hb / 2 + slack
    sl = slice(123456789, 123456789 + (1 << 20))
    _, _, rq = fo.quantize(np.concatenate([w[sl].cpu().numpy(), [w.min().item(), w.max().item()]]))
    assert np.array_equal(q[sl].cpu().numpy(), rq[:-2])


# ------------------------------------------------------------------ K5


def test_hash_matches_reference():
    g = load("hash")
    pairs = [(str(f), str(t)) for f, t in zip(g["fields"], g["tokens"])]
    bits = g["bits"]
    items = [f.encode() + b"\x1f" + t.encode() for f, t in pairs]
    blob, off = hashing.pack_strings(items)
    raw = hashing.hash_bytes(blob, off, 32, DEV).cpu().numpy()
    got = raw & ((1 << bits.astype(np.int64)) - 1)
    assert (got == g["out"]).all()
    rb, ro = hashing.pack_strings([bytes(x) for x in g["raw"]])
    assert (hashing.hash_bytes(rb, ro, 32, DEV).cpu().numpy() == g["raw_out"]).all()
    h = hashing.hash_features([("user", "u_42"), ("ad", "u_42")], 18, DEV).cpu().tolist()
    assert h[0] != h[1] and h == [fo.hash_feature("user", "u_42", 18),
                                  fo.hash_feature("ad", "u_42", 18)]
    with pytest.raises(ContractError):
        hashing.hash_features([("a", "b")], 9, DEV)


def test_hash_synthetic_ranks_large_batch():
    """1M (field, rank) tokens hashed on the GPU == the vectorised generator."""
    rng = np.random.default_rng(5)
    fr = rng.integers(0, 40, 1 << 20)
    rr = rng.integers(1, 1 << 25, 1 << 20)
    items = [f"f{f}".encode() + b"\x1f" + f"t{r}".encode() for f, r in zip(fr, rr)]
    blob, off = hashing.pack_strings(items)
    got = hashing.hash_bytes(blob, off, 25, DEV).cpu().numpy()
    ref = synth.hash_ranks(torch.as_tensor(fr), torch.as_tensor(rr), 25).numpy()
    assert (got == ref).all()


# ------------------------------------------------------------------ K3


def _ctx_mode(ctx_mlp, monkeypatch):
    if ctx_mlp == "ring":  # default: K3 v2 (row ring + tcgen05 MLP) where it applies
        monkeypatch.delenv("DFFM_CTX_MLP", raising=False)
    else:
        monkeypatch.setenv("DFFM_CTX_MLP", ctx_mlp)


@pytest.mark.parametrize("ctx_mlp", ["simt", "tc", "ring"])
def test_context_cache_matches_reference_merged_forward(ctx_mlp, monkeypatch):
    _ctx_mode(ctx_mlp, monkeypatch)
    g = load("ctx")
    F, k, hidden, bits, flat = fixture_flat(g)
    cfg = ModelConfig(n_fields=F, k=k, hidden_sizes=hidden, hash_bits=bits)
    st = WeightStore.from_flat(cfg, flat, DEV, with_optimizer=False)
    p = inference.score_requests(g["ctx_idx"], g["ctx_val"], g["cand_idx"], g["cand_val"], st)
    assert np.abs(p.double().cpu().numpy() - g["prob"]).max() <= 1e-6
    # per-request API with staleness
    cache = inference.build_context_cache(g["ctx_idx"][3], g["ctx_val"][3], st)
    p3 = inference.predict_batch(cache, g["cand_idx"][3], g["cand_val"][3], st)
    assert np.abs(p3.double().cpu().numpy() - g["prob"][3]).max() <= 1e-6
    st.mark_mutated()
    with pytest.raises(StaleCacheError):
        inference.predict_batch(cache, g["cand_idx"][3], g["cand_val"][3], st)


@pytest.mark.parametrize("ctx_mlp", ["simt", "tc", "ring"])
def test_context_cache_equals_uncached_forward_u16(ctx_mlp, monkeypatch):
    """K3 (SIMT, staged tensor-core MLP, or the row-ring K3 v2) == K1 on the
    merged examples == oracle."""
    _ctx_mode(ctx_mlp, monkeypatch)
    wl = configs.CFG4
    bits = 14
    ost = fo.random_store(24, 8, (64, 32), bits, seed=44)
    cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    sq, _ = quant.quantize_store(st)
    R, C = 37, 101
    ci, cv = synth.make_examples(wl, R, seed=1, hash_bits=bits, n_fields=16)
    di, dv = synth.make_examples(wl, R * C, seed=2, hash_bits=bits, field_offset=16, n_fields=8)
    di, dv = di.view(R, C, 8, 1), dv.view(R, C, 8, 1)
    p = inference.score_requests(ci, cv, di, dv, sq).cpu().numpy()
    merged_i = torch.cat([ci[:, None].expand(R, C, 16, 1), di], 2).reshape(R * C, 24, 1)
    merged_v = torch.cat([cv[:, None].expand(R, C, 16, 1), dv], 2).reshape(R * C, 24, 1)
    p_unc = predict_batch(merged_i, merged_v, sq).cpu().numpy().reshape(R, C)
    assert np.abs(p - p_unc).max() <= 1e-6
    cst, ridx, _ = compact_oracle(sq, merged_i.numpy())
    _, ref = fo.forward_batch(ridx, merged_v.numpy(), cst)
    assert np.abs(p.reshape(-1) - ref).max() <= 1e-6


@pytest.mark.parametrize("wdtype,Mc,Md,C,Fc,Fd", [
    ("f32", 2, 2, 40, 10, 6), ("bf16", 1, 3, 33, 10, 6),  # C < 64: K3 v1
    ("u16", 3, 1, 64, 10, 6),    # ring, bundles of 4, several chunks per pair warp
    ("f32", 2, 2, 72, 10, 6),    # ring, 2 slots per candidate field, bundles of 2
    ("bf16", 1, 3, 65, 10, 6),   # ring, 3 slots per candidate field, odd C: no bundling
    ("u16", 2, 1, 96, 16, 8),    # ring, cfg4 field split: one chunk per pair warp (register-resident context segments), bundles of 4
    ("f32", 1, 1, 66, 16, 8),    # the same path, bundles of 2
])
def test_context_ring_edge_cases_match_oracle(wdtype, Mc, Md, C, Fc, Fd, monkeypatch):
    """K3 v2 with multi-slot context and candidate fields, absent context and
    candidate fields, empty candidates; every table dtype and every bundle size;
    vs the oracle."""
    monkeypatch.delenv("DFFM_CTX_MLP", raising=False)
    bits = 12
    F = Fc + Fd
    ost = fo.random_store(F, 8, (32, 16), bits, seed=Mc * 10 + Md)
    cfg = ModelConfig(n_fields=F, k=8, hidden_sizes=(32, 16), hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    if wdtype == "bf16":
        st = WeightStore.from_flat(cfg, ost.flat(False), DEV, "bf16", False)
    elif wdtype == "u16":
        st, _ = quant.quantize_store(st)
    rng = np.random.default_rng(Mc + 7 * Md)
    R = 21

    def slots(shape, M):
        idx = rng.integers(-1, 1 << bits, size=shape + (M,)).astype(np.int32)
        idx = np.sort(np.where(idx < 0, np.iinfo(np.int32).max, idx), axis=-1)
        idx = np.where(idx == np.iinfo(np.int32).max, -1, idx)
        flat = idx.reshape(-1, M)
        for r in range(len(flat)):
            live = np.unique(flat[r][flat[r] >= 0])
            flat[r] = -1
            flat[r][:len(live)] = live
        return flat.reshape(idx.shape)

    ci = slots((R, Fc), Mc)
    ci[2] = -1  # a request without context features
    di = slots((R, C, Fd), Md)
    di[:, ::7] = -1  # empty candidates
    di[:, 1::5, Fd // 2] = -1  # an absent candidate field
    ci[4, Fc // 3] = -1  # an absent context field
    cv = np.where(ci >= 0, rng.lognormal(size=ci.shape), 0).astype(np.float32)
    dv = np.where(di >= 0, rng.lognormal(size=di.shape), 0).astype(np.float32)
    p = inference.score_requests(ci, cv, di, dv, st).cpu().numpy()
    M = max(Mc, Md)
    mi = np.full((R, C, F, M), -1, np.int32)
    mv = np.zeros((R, C, F, M), np.float32)
    mi[:, :, :Fc, :Mc] = ci[:, None]
    mv[:, :, :Fc, :Mc] = cv[:, None]
    mi[:, :, Fc:, :Md] = di
    mv[:, :, Fc:, :Md] = dv
    cst, ridx, _ = compact_oracle(st, mi.reshape(R * C, F, M))
    _, ref = fo.forward_batch(ridx, mv.reshape(R * C, F, M), cst)
    assert np.abs(p.reshape(-1) - ref).max() <= 1e-6


def test_context_ring_bad_context_index_is_contract_error(monkeypatch):
    """K3 v2: an out-of-range context bucket raises ContractError (reported at
    the request's first candidate)."""
    monkeypatch.delenv("DFFM_CTX_MLP", raising=False)
    bits = 10
    ost = fo.random_store(12, 8, (16,), bits, seed=3)
    cfg = ModelConfig(n_fields=12, k=8, hidden_sizes=(16,), hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    R, C = 5, 64
    rng = np.random.default_rng(0)
    ci = rng.integers(0, 1 << bits, size=(R, 8, 1)).astype(np.int32)
    di = rng.integers(0, 1 << bits, size=(R, C, 4, 1)).astype(np.int32)
    ci[3, 2, 0] = 1 << bits  # out of range
    with pytest.raises(ContractError):
        inference.score_requests(ci, np.ones_like(ci, np.float32), di,
                                 np.ones_like(di, np.float32), st)


def test_prebuilt_context_cache_is_reused_without_a_context_pass():
    """build_context_cache runs the context pass once (dffm_ctx_build);
    predict_batch(cache, ...) scores against the device-resident blob with no
    context build (library build counter unchanged), bit-identical to the
    in-kernel build of score_requests; ContextCacheMap dedupes repeated
    contexts by their digest and drops entries on a version bump."""
    from paper_2407_10115_b200 import _lib
    F, Fc, k, bits, C = 24, 16, 8, 12, 96
    ost = fo.random_store(F, k, (64, 32), bits, seed=21)
    cfg = ModelConfig(n_fields=F, k=k, hidden_sizes=(64, 32), hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    rng = np.random.default_rng(5)
    ci = rng.integers(0, 1 << bits, (3, Fc, 1)).astype(np.int32)
    cv = np.ones_like(ci, np.float32)
    di = rng.integers(0, 1 << bits, (3, C, F - Fc, 1)).astype(np.int32)
    dv = rng.lognormal(size=di.shape).astype(np.float32)
    ref = inference.score_requests(ci, cv, di, dv, st).cpu().numpy()
    lib = _lib.lib()
    cache = inference.build_context_cache(ci[1], cv[1], st)
    n0 = lib.dffm_ctx_build_count()
    p1 = inference.predict_batch(cache, di[1], dv[1], st).cpu().numpy()
    p2 = inference.predict_batch(cache, di[1], dv[1], st).cpu().numpy()
    assert lib.dffm_ctx_build_count() == n0  # no context pass on the cached path
    assert np.array_equal(p1, ref[1]) and np.array_equal(p2, ref[1])
    # digest map: the same context (same triples, padded differently) is built once
    cmap = inference.ContextCacheMap(st)
    a = cmap.get(ci[0], cv[0])
    pad_i = np.concatenate([ci[0], np.full_like(ci[0], -1)], axis=1)
    pad_v = np.concatenate([cv[0], np.zeros_like(cv[0])], axis=1)
    assert inference._digest(pad_i, pad_v) == a.digest
    b = cmap.get(ci[0].copy(), cv[0].copy())
    assert cmap.misses == 1 and cmap.hits == 1 and a is b
    st.mark_mutated()
    c = cmap.get(ci[0], cv[0])
    assert c is not a and c.store_version == st.version
    # bad context index -> ContractError at build time
    bad = ci[0].copy()
    bad[3, 0] = 1 << (bits + 2)
    with pytest.raises(ContractError):
        inference.build_context_cache(bad, cv[0], st)


def test_host_request_scorer_matches_device_path_and_reports_global_candidate():
    """inference.HostRequestScorer (pinned host requests, chunked over three streams)
    returns the bits of score_requests on device tensors; a bad candidate bucket in
    a later chunk raises ContractError at its stream-global candidate number."""
    bits = 12
    F, Fc, C = 24, 16, 68
    ost = fo.random_store(F, 8, (64, 32), bits, seed=9)
    cfg = ModelConfig(n_fields=F, k=8, hidden_sizes=(64, 32), hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, with_optimizer=False)
    rng = np.random.default_rng(11)
    R = 50
    ci = torch.from_numpy(rng.integers(0, 1 << bits, (R, Fc, 1)).astype(np.int32)).pin_memory()
    cv = torch.ones((R, Fc, 1)).pin_memory()
    di = torch.from_numpy(rng.integers(0, 1 << bits, (R, C, F - Fc, 1)).astype(np.int32)).pin_memory()
    dv = torch.from_numpy(rng.lognormal(size=(R, C, F - Fc, 1)).astype(np.float32)).pin_memory()
    ref = inference.score_requests(ci, cv, di, dv, st).cpu()
    hs = inference.HostRequestScorer(st, Fc, 1, C, 1, chunk_requests=12)
    out = torch.empty((R, C)).pin_memory()
    hs(ci, cv, di, dv, out)
    assert torch.equal(out, ref)
    hs(ci, cv, di, dv, out)  # reusable
    assert torch.equal(out, ref)
    di[31, 5, 2, 0] = 1 << bits
    with pytest.raises(ContractError) as ei:
        hs(ci, cv, di, dv, out)
    assert ei.value.example == 31 * C + 5
