"""K1 fused forward parity (GPU) against the reference goldens and the oracle.

Tolerance: predictions within 1e-5 relative (BASELINE north star, fp32); the
kernel accumulates pair dots in f32 and the lr / pair sums / MergeNorm
statistics in f64."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200 import configs, synth
from paper_2407_10115_b200.errors import ContractError, NumericError
from paper_2407_10115_b200.model import ModelConfig, WeightStore, predict_batch
from tests.golden_io import fixture_flat, load
from tests.remap import compact_oracle, rel_err

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
RTOL = 1e-5


def store_from_oracle(ost, wdtype="f32", with_optimizer=False):
    cfg = ModelConfig(n_fields=ost.n_fields, k=ost.k, hidden_sizes=ost.hidden_sizes,
                      hash_bits=ost.hash_bits)
    return WeightStore.from_flat(cfg, ost.flat(False), DEV, wdtype, with_optimizer)


@pytest.mark.parametrize("name,wdtype", [("cfg1", "f32"), ("cfg2", "f32"), ("cfg5", "bf16"),
                                         ("cfg5", "f32")])
def test_forward_matches_reference_golden(name, wdtype):
    g = load(f"fwd_{name}")
    F, k, hidden, bits, flat = fixture_flat(g)
    cfg = ModelConfig(n_fields=F, k=k, hidden_sizes=hidden, hash_bits=bits)
    st = WeightStore.from_flat(cfg, flat, DEV, wdtype, with_optimizer=False)
    lg = torch.empty(g["idx"].shape[0], device=DEV)
    p = predict_batch(g["idx"], g["val"], st, logits=lg).double().cpu().numpy()
    assert rel_err(p, g["prob"]).max() < RTOL
    np.testing.assert_allclose(lg.double().cpu().numpy(), g["logit"], rtol=1e-5, atol=2e-6)


CASES = [
    # F, k, hidden, M, bits, n
    (8, 4, (), 1, 10, 1000),
    (24, 8, (64, 32), 3, 12, 777),
    (24, 8, (64, 32), 1, 12, 300),
    (5, 3, (7,), 2, 8, 129),          # runtime-k path, hidden not a multiple of 4
    (3, 1, (4, 4, 4, 4), 6, 6, 70),   # k=1, 4 hidden layers, M > 4 (generic slot loop)
    (1, 2, (3,), 2, 5, 33),           # F=1: P=0, MergeNorm of one value
    (2, 16, (), 2, 7, 65),
    (12, 32, (16,), 2, 9, 64),
    (40, 16, (256, 128), 1, 11, 200),
]


@pytest.mark.parametrize("F,k,hidden,M,bits,n", CASES)
def test_forward_matches_oracle(F, k, hidden, M, bits, n):
    rng = np.random.default_rng(F * 1000 + k)
    ost = fo.random_store(F, k, hidden, bits, seed=F + k)
    idx = rng.integers(-1, 1 << bits, size=(n, F, M)).astype(np.int32)
    idx = np.sort(np.where(idx < 0, np.iinfo(np.int32).max, idx), axis=2)
    idx = np.where(idx == np.iinfo(np.int32).max, -1, idx)
    for e in range(n):  # canonical: unique within a field
        for f in range(F):
            row = idx[e, f]
            live = np.unique(row[row >= 0])
            idx[e, f] = -1
            idx[e, f, :len(live)] = live
    val = np.where(idx >= 0, rng.lognormal(size=idx.shape), 0).astype(np.float32)
    st = store_from_oracle(ost)
    p = predict_batch(idx, val, st).double().cpu().numpy()
    _, ref = fo.forward_batch(idx, val, ost)
    assert rel_err(p, ref).max() < RTOL


@pytest.mark.parametrize("family", [1, 2, 5])
@pytest.mark.parametrize("wdtype", ["f32", "bf16", "u16"])
def test_every_forward_family_matches_oracle(family, wdtype):
    """Every K1 kernel family (1 warp-specialised fused, 2 CTA-synchronous,
    5 row-ring gather + tcgen05 3xTF32 MLP) on cfg2-shaped inputs and every
    table storage type."""
    from paper_2407_10115_b200 import _lib
    from paper_2407_10115_b200.quant import quantize_store
    wl = configs.CFG2
    ost = fo.random_store(24, 8, (64, 32), 12, seed=4)
    idx, val = synth.make_examples(wl, 1537, seed=8, hash_bits=12)
    st = store_from_oracle(ost)
    if wdtype == "bf16":
        st = WeightStore.from_flat(st.config, ost.flat(False), DEV, "bf16", False)
    elif wdtype == "u16":
        st, _ = quantize_store(st)
    _lib.check(_lib.lib().dffm_set_forward_family(family))
    try:
        p = predict_batch(idx, val, st).double().cpu().numpy()
    finally:
        _lib.lib().dffm_set_forward_family(-1)
    cst, ridx, _ = compact_oracle(st, idx.numpy())
    _, ref = fo.forward_batch(ridx, val.numpy(), cst)
    assert rel_err(p, ref).max() < RTOL


@pytest.mark.parametrize("family", [-1, 5, 1])
@pytest.mark.parametrize("n", [1, 127, 300])
def test_forward_cfg5_shape_tensor_core_mlp(family, n):
    """cfg5 shape (F=40, k=16, bf16 tables, MLP 781-256-128-1): the default
    dispatch picks the tcgen05 MLP; ragged tails (n % 128 != 0) included."""
    from paper_2407_10115_b200 import _lib
    wl = configs.CFG5
    ost = fo.random_store(40, 16, (256, 128), 12, seed=5, scale=0.05)
    idx, val = synth.make_examples(wl, n, seed=11, hash_bits=12)
    st = WeightStore.from_flat(ModelConfig(n_fields=40, k=16, hidden_sizes=(256, 128),
                                           hash_bits=12), ost.flat(False), DEV, "bf16", False)
    _lib.check(_lib.lib().dffm_set_forward_family(family))
    try:
        lg = torch.empty(n, device=DEV)
        p = predict_batch(idx, val, st, logits=lg).double().cpu().numpy()
    finally:
        _lib.lib().dffm_set_forward_family(-1)
    cst, ridx, _ = compact_oracle(st, idx.numpy())
    lref, ref = fo.forward_batch(ridx, val.numpy(), cst)
    assert rel_err(p, ref).max() < RTOL
    np.testing.assert_allclose(lg.double().cpu().numpy(), lref, rtol=1e-5, atol=1e-5)


def test_forward_tc_slices_and_nonfinite_nn():
    """Several staging slices (DFFM_TC_SLICE is 32*148*128 rows by default) and
    a non-finite hidden unit reported as block "nn" at the first example."""
    from paper_2407_10115_b200 import _lib
    ost = fo.random_store(8, 4, (32, 16), 10, seed=3)
    n = 32 * 148 * 128 * 2 + 77
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 1 << 10, size=(n, 8, 1)).astype(np.int32)
    val = np.ones_like(idx, dtype=np.float32)
    st = store_from_oracle(ost)
    _lib.check(_lib.lib().dffm_set_forward_family(5))
    try:
        p = predict_batch(idx, val, st).double().cpu().numpy()
        sel = np.r_[0:64, n - 200:n]
        _, ref = fo.forward_batch(idx[sel], val[sel], ost)
        assert rel_err(p[sel], ref).max() < RTOL
        o = ost.copy()
        o.layers[1][0][:, 5] = np.inf
        with pytest.raises(NumericError) as ei:
            predict_batch(idx, val, store_from_oracle(o))
        assert ei.value.example == 0 and ei.value.block == "nn"
    finally:
        _lib.lib().dffm_set_forward_family(-1)


def test_forward_bf16_and_u16_tables_match_widened_oracle():
    from paper_2407_10115_b200.quant import quantize_store
    wl = configs.CFG2
    ost = fo.random_store(24, 8, (64, 32), 12, seed=4)
    idx, val = synth.make_examples(wl, 2000, seed=8, hash_bits=12)
    st = store_from_oracle(ost)
    for variant in ("bf16", "u16"):
        if variant == "bf16":
            s2 = WeightStore.from_flat(st.config, ost.flat(False), DEV, "bf16", False)
        else:
            s2, _ = quantize_store(st)
        p = predict_batch(idx, val, s2).double().cpu().numpy()
        cst, ridx, _ = compact_oracle(s2, idx.numpy())
        _, ref = fo.forward_batch(ridx, val.numpy(), cst)
        assert rel_err(p, ref).max() < RTOL, variant


def test_forward_empty_and_ragged_batches():
    ost = fo.random_store(6, 8, (8,), 8, seed=1)
    st = store_from_oracle(ost)
    out = predict_batch(np.zeros((0, 6, 2), np.int32), np.zeros((0, 6, 2), np.float32), st)
    assert out.numel() == 0
    for n in (1, 31, 33, 257):
        idx = np.full((n, 6, 2), -1, np.int32)
        idx[:, :, 0] = np.arange(n * 6).reshape(n, 6) % 256
        val = (idx >= 0).astype(np.float32)
        p = predict_batch(idx, val, st).double().cpu().numpy()
        _, ref = fo.forward_batch(idx, val, ost)
        assert rel_err(p, ref).max() < RTOL


def test_forward_nonfinite_reports_first_example_and_block():
    ost = fo.random_store(4, 4, (8,), 6, seed=2)
    idx = np.full((50, 4, 1), -1, np.int32)
    idx[:, 0, 0] = 1
    idx[:, 1, 0] = 2
    val = (idx >= 0).astype(np.float32)
    cases = []
    o = ost.copy(); o.ffm[9, 2, 0] = np.inf; cases.append((o, 9, 1, "ffm"))   # noqa: E702
    o = ost.copy(); o.lr[11] = np.nan; cases.append((o, 11, 3, "lr"))          # noqa: E702
    for o, bucket, field, block in cases:
        ix = idx.copy()
        ix[17, field, 0] = bucket
        ix[33, field, 0] = bucket
        if block == "ffm":
            ix[17, 2, 0] = 5  # the pair (field 1, field 2) reads ffm[9][2]
            ix[33, 2, 0] = 5
        st = store_from_oracle(o)
        with pytest.raises(NumericError) as ei:
            predict_batch(ix, (ix >= 0).astype(np.float32), st)
        assert ei.value.example == 17 and ei.value.block == block
        with pytest.raises(fo.OracleNumericError) as eo:
            fo.forward(fo.row_to_fields(ix[17], (ix[17] >= 0).astype(np.float32)), o)
        assert eo.value.block == block
    o = ost.copy()
    o.layers[0][0][:, 3] = np.inf
    st = store_from_oracle(o)
    with pytest.raises(NumericError) as ei:
        predict_batch(idx, val, st)
    assert ei.value.example == 0 and ei.value.block == "nn"


def test_forward_out_of_range_index_is_contract_error():
    ost = fo.random_store(3, 4, (), 6, seed=2)
    st = store_from_oracle(ost)
    idx = np.zeros((4, 3, 1), np.int32)
    idx[2, 1, 0] = 64
    with pytest.raises(ContractError):
        predict_batch(idx, np.ones_like(idx, dtype=np.float32), st)


@pytest.mark.slow
def test_forward_cfg2_full_table_sample():
    """BASELINE cfg2 at full size (2^24 buckets, 1M batch): oracle on a sample."""
    wl = configs.CFG2
    cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=24)
    st = WeightStore(cfg, DEV, with_optimizer=False)
    gen = torch.Generator(device=DEV).manual_seed(wl.weight_seed)
    st.lr.copy_(synth.normal_table(st.lr.numel(), 0.05, gen, DEV))
    st.ffm.view(-1).copy_(synth.normal_table(st.ffm.numel(), 0.05, gen, DEV))
    for w, b in st.nn_layers:
        w.copy_(torch.randn(w.shape, generator=gen, device=DEV) * 0.05)
        b.copy_(torch.randn(b.shape, generator=gen, device=DEV) * 0.05)
    idx, val = synth.make_examples(wl, 1 << 20, device=DEV)
    p = predict_batch(idx, val, st)
    assert torch.isfinite(p).all()
    sel = torch.randperm(1 << 20, generator=torch.Generator().manual_seed(0))[:4096]
    si = idx[sel.to(DEV)].cpu().numpy()
    sv = val[sel.to(DEV)].cpu().numpy()
    cst, ridx, _ = compact_oracle(st, si)
    _, ref = fo.forward_batch(ridx, sv, cst)
    assert rel_err(p[sel.to(DEV)].double().cpu().numpy(), ref).max() < RTOL
    # size-independent property: permuting the batch permutes the outputs exactly
    perm = torch.randperm(1 << 20, device=DEV)
    p2 = predict_batch(idx[perm], val[perm], st)
    assert torch.equal(p2, p[perm])


def _full_store(wl):
    """Seeded on-device table of the workload's full size (as bench.build_store)."""
    cfg = ModelConfig(n_fields=wl.n_fields, k=wl.k, hidden_sizes=wl.hidden, hash_bits=wl.hash_bits)
    st = WeightStore(cfg, DEV, "bf16" if wl.weight_dtype == "bf16" else "f32",
                     with_optimizer=False)
    gen = torch.Generator(device=DEV).manual_seed(wl.weight_seed)
    for t in (st.lr, st.ffm):
        flat = t.view(-1)
        for c0 in range(0, flat.numel(), 1 << 28):
            c1 = min(flat.numel(), c0 + (1 << 28))
            flat[c0:c1].copy_(torch.randn(c1 - c0, generator=gen, device=DEV) * wl.weight_scale)
    for w, b in st.nn_layers:
        w.copy_(torch.randn(w.shape, generator=gen, device=DEV) * wl.weight_scale)
        b.copy_(torch.randn(b.shape, generator=gen, device=DEV) * wl.weight_scale)
    return st


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg1", "cfg5"])
def test_forward_full_size_config_sample(name):
    """BASELINE cfg1 (whole 65,536 batch) and cfg5 (2^25 buckets, 43 GB bf16
    table, 8,388,608 examples; 4,096 sampled) against the oracle."""
    wl = {"cfg1": configs.CFG1, "cfg5": configs.CFG5}[name]
    st = _full_store(wl)
    cdf = synth.zipf_cdf(1 << wl.hash_bits, wl.zipf_alpha, DEV) if wl.dist == "zipf" else None
    idx, val = synth.make_examples(wl, wl.n_examples, device=DEV, cdf=cdf)
    del cdf
    p = predict_batch(idx, val, st)
    assert torch.isfinite(p).all()
    n = idx.shape[0]
    sel = torch.randperm(n, generator=torch.Generator().manual_seed(1))[: min(n, 4096)]
    si, sv = idx[sel.to(DEV)].cpu().numpy(), val[sel.to(DEV)].cpu().numpy()
    cst, ridx, _ = compact_oracle(st, si)
    _, ref = fo.forward_batch(ridx, sv, cst)
    assert rel_err(p[sel.to(DEV)].double().cpu().numpy(), ref).max() < RTOL


@pytest.mark.slow
def test_context_cache_full_size_cfg4_sample():
    """BASELINE cfg4 at full size: u16-quantised 2^24 tables, 2,000 requests x
    500 candidates through K3; 4,096 sampled candidates vs the oracle on the
    merged examples."""
    from paper_2407_10115_b200 import inference
    from paper_2407_10115_b200.quant import quantize_store
    wl = configs.CFG4
    st, _ = quantize_store(_full_store(wl))
    torch.cuda.empty_cache()
    R, C, Fc = wl.n_requests, wl.n_candidates, wl.ctx_fields
    cdf = synth.zipf_cdf(1 << wl.hash_bits, wl.zipf_alpha, DEV)
    ci, cv = synth.make_examples(wl, R, seed=wl.data_seed, device=DEV, cdf=cdf, n_fields=Fc)
    di, dv = synth.make_examples(wl, R * C, seed=wl.data_seed + 1, device=DEV, cdf=cdf,
                                 n_fields=wl.n_fields - Fc, field_offset=Fc)
    di, dv = di.view(R, C, wl.n_fields - Fc, -1), dv.view(R, C, wl.n_fields - Fc, -1)
    p = inference.score_requests(ci, cv, di, dv, st)
    g = torch.Generator().manual_seed(2)
    rr = torch.randint(0, R, (4096,), generator=g)
    cc = torch.randint(0, C, (4096,), generator=g)
    mi = torch.cat([ci[rr.to(DEV)], di[rr.to(DEV), cc.to(DEV)]], 1).cpu().numpy()
    mv = torch.cat([cv[rr.to(DEV)], dv[rr.to(DEV), cc.to(DEV)]], 1).cpu().numpy()
    cst, ridx, _ = compact_oracle(st, mi)
    _, ref = fo.forward_batch(ridx, mv, cst)
    got = p[rr.to(DEV), cc.to(DEV)].double().cpu().numpy()
    assert rel_err(got, ref).max() < RTOL


RING_CASES = [
    # F, k, hidden, M, bits, n, wdtype
    (24, 8, (64, 32), 3, 12, 1000, "f32"),
    (8, 4, (32, 16), 4, 10, 513, "f32"),
    (40, 16, (256, 128), 1, 11, 300, "bf16"),
    (16, 16, (64,), 2, 10, 257, "u16"),
    (32, 8, (128, 64), 4, 10, 200, "f32"),   # F*M = 128 slots (the kernel's maximum)
    (2, 8, (16,), 2, 6, 90, "bf16"),          # P = 1: one pair chunk per example
]


@pytest.mark.parametrize("F,k,hidden,M,bits,n,wdtype", RING_CASES)
def test_forward_row_ring_gather_matches_oracle(F, k, hidden, M, bits, n, wdtype):
    """K1 v8 (warp-specialised circular row ring feeding the tcgen05 MLP,
    forward_rsw.cuh): ragged multi-slot fields, fully empty examples (no rows
    allocated), every table dtype, against the oracle."""
    from paper_2407_10115_b200 import _lib
    from paper_2407_10115_b200.quant import quantize_store
    rng = np.random.default_rng(F * 7919 + M)
    ost = fo.random_store(F, k, hidden, bits, seed=F + M)
    idx = rng.integers(-1, 1 << bits, size=(n, F, M)).astype(np.int32)
    idx = np.sort(np.where(idx < 0, np.iinfo(np.int32).max, idx), axis=2)
    idx = np.where(idx == np.iinfo(np.int32).max, -1, idx)
    for e in range(n):
        for f in range(F):
            live = np.unique(idx[e, f][idx[e, f] >= 0])
            idx[e, f] = -1
            idx[e, f, :len(live)] = live
    idx[::11] = -1      # empty examples
    idx[5::13, 1:] = -1  # one present field
    val = np.where(idx >= 0, rng.lognormal(size=idx.shape), 0).astype(np.float32)
    st = store_from_oracle(ost)
    if wdtype == "bf16":
        st = WeightStore.from_flat(st.config, ost.flat(False), DEV, "bf16", False)
    elif wdtype == "u16":
        st, _ = quantize_store(st)
    _lib.check(_lib.lib().dffm_set_forward_family(5))
    try:
        lg = torch.empty(n, device=DEV)
        p = predict_batch(idx, val, st, logits=lg).double().cpu().numpy()
    finally:
        _lib.lib().dffm_set_forward_family(-1)
    cst, ridx, _ = compact_oracle(st, idx)
    lref, ref = fo.forward_batch(ridx, val, cst)
    assert rel_err(p, ref).max() < RTOL
    np.testing.assert_allclose(lg.double().cpu().numpy(), lref, rtol=1e-5, atol=1e-5)


def test_forward_row_ring_nonfinite_and_bad_index():
    """Row-ring gather: the first non-finite example/block and a bad bucket
    index (ContractError) are reported like the reference loop would."""
    from paper_2407_10115_b200 import _lib
    ost = fo.random_store(4, 4, (16,), 6, seed=2)
    idx = np.full((300, 4, 2), -1, np.int32)
    idx[:, 0, 0] = 1
    idx[:, 1, 0] = 2
    idx[:, 2, 0] = 5
    o = ost.copy()
    o.ffm[9, 2, 0] = np.inf
    ix = idx.copy()
    ix[170, 1, 1] = 9
    ix[233, 1, 1] = 9
    _lib.check(_lib.lib().dffm_set_forward_family(5))
    try:
        with pytest.raises(NumericError) as ei:
            predict_batch(ix, (ix >= 0).astype(np.float32), store_from_oracle(o))
        assert ei.value.example == 170 and ei.value.block == "ffm"
        ix = idx.copy()
        ix[77, 3, 0] = 1 << 6
        with pytest.raises(ContractError):
            predict_batch(ix, (ix >= 0).astype(np.float32), store_from_oracle(ost))
    finally:
        _lib.lib().dffm_set_forward_family(-1)


@pytest.mark.parametrize("cfgname", ["cfg2", "cfg5"])
def test_forward_is_bit_reproducible_across_launches(cfgname):
    """Race detector for the warp-specialised row ring and the tcgen05 MLP: the same
    batch scored four times (hot and cold L2, the ring and the TMEM regions in
    different phases) gives identical bits; so do the seeded inputs when they are
    generated twice (the Zipf CDF is summed on the host)."""
    wl = {"cfg2": configs.CFG2, "cfg5": configs.CFG5}[cfgname]
    bits = 16
    F, k, M = wl.n_fields, wl.k, wl.max_per_field
    ost = fo.random_store(F, k, tuple(wl.hidden), bits, seed=3)
    st = store_from_oracle(ost, "bf16" if cfgname == "cfg5" else "f32")
    n = 150_000
    idx, val = synth.make_examples(wl, n, seed=5, device=DEV, hash_bits=bits)
    idx2, val2 = synth.make_examples(wl, n, seed=5, device=DEV, hash_bits=bits)
    assert torch.equal(idx, idx2) and torch.equal(val, val2)
    ref = predict_batch(idx, val, st).clone()
    flush = torch.empty(160 << 20, dtype=torch.uint8, device=DEV)
    for r in range(3):
        if r & 1:
            flush.zero_()
        p = predict_batch(idx, val, st)
        assert torch.equal(p, ref), f"launch {r}: {(p != ref).sum().item()} examples differ"
