"""Host-side logic on CPU: config validation, packing, flat layout,
serialisation byte-identity, metrics, synthetic generator -- all checked
against reference-generated goldens (no GPU)."""

import numpy as np
import pytest
import torch

from paper_2407_10115_b200 import configs, features, metrics, synth
from paper_2407_10115_b200.errors import ContractError, FormatError
from paper_2407_10115_b200.model import (ModelConfig, WeightStore, flat_weight_view, init_model,
                                         pair_position, store_from_bytes)
from tests.golden_io import load

CPU = torch.device("cpu")


def test_model_config_contract():
    for bad in [dict(n_fields=0), dict(n_fields=2, k=0), dict(n_fields=2, hidden_sizes=(1,) * 5),
                dict(n_fields=2, lr_ffm=0), dict(n_fields=2, power_t=1.5),
                dict(n_fields=2, hash_bits=30)]:
        with pytest.raises(ContractError):
            ModelConfig(**bad)
    c = ModelConfig(n_fields=3, k=2, hidden_sizes=[4])
    assert ModelConfig.from_json(c.to_json()) == c
    with pytest.raises(FormatError):
        ModelConfig.from_json("{nope")


def test_pair_position_matches_reference_order():
    pos = pair_position(4)
    assert pos[0, 1] == 0 and pos[0, 3] == 2 and pos[1, 2] == 3 and pos[2, 3] == 5
    assert pos[3, 2] == 5 and pos[1, 1] == -1


def test_flat_weight_view_byte_identical_to_reference():
    g = load("serial")
    cfg = ModelConfig.from_json(str(g["cfg_json"]))
    st = init_model(cfg, device=CPU)  # chunked replica of M:233-272
    full = flat_weight_view(st, True)
    infer = flat_weight_view(st, False)
    assert full == g["full"].tobytes()
    assert infer == g["infer"].tobytes()
    back = store_from_bytes(full, device=CPU)
    assert flat_weight_view(back, True) == full  # S:149 round trip
    back2 = store_from_bytes(infer, device=CPU)
    assert (back2.lr_acc == 1).all()  # M:682-683
    with pytest.raises(FormatError):
        store_from_bytes(b"XXXX" + full[4:], device=CPU)
    with pytest.raises(FormatError):
        store_from_bytes(full[:-4], device=CPU)


def test_init_model_chunking_invariant():
    cfg = ModelConfig(n_fields=3, k=2, hidden_sizes=(4,), hash_bits=6, init_seed=9)
    a = init_model(cfg, device=CPU, chunk=7).weight_values()
    b = init_model(cfg, device=CPU, chunk=1 << 20).weight_values()
    assert a.tobytes() == b.tobytes()


def test_store_layout_and_single_weight_offset():
    # stores differing in one weight differ in exactly 4 bytes at the documented offset
    cfg = ModelConfig(n_fields=3, k=2, hidden_sizes=(4,), hash_bits=5)
    a = WeightStore(cfg, CPU)
    b = a.copy()
    b.ffm[7, 2, 1] = 1.5
    fa, fb = flat_weight_view(a), flat_weight_view(b)
    diff = [i for i in range(len(fa)) if fa[i] != fb[i]]
    hdr = len(fa) - 4 * a.total_slots
    off = hdr + 4 * (a.ffm_offset if hasattr(a, "ffm_offset") else a.lr_size) + 4 * ((7 * 3 + 2) * 2 + 1)
    assert diff and min(diff) >= off and max(diff) < off + 4


def test_pack_examples_canonicalises():
    class FF:
        def __init__(self, f, i, v):
            self.field_id, self.indices, self.values = f, np.array(i), np.array(v, float)

    class Ex:
        def __init__(self, label, fields):
            self.label, self.fields = label, fields

    exs = [Ex(1, [FF(2, [5, 3], [1.0, 2.0]), FF(0, [9], [0.5]), FF(2, [5], [4.0])]), Ex(0, [])]
    idx, val, lab = features.pack_examples(exs, 3)
    assert idx.shape == (2, 3, 2)
    assert idx[0, 2].tolist() == [3, 5] and val[0, 2].tolist() == [2.0, 5.0]
    assert idx[0, 0].tolist() == [9, -1] and idx[0, 1].tolist() == [-1, -1]
    assert (idx[1] == -1).all() and lab.tolist() == [1, 0]
    with pytest.raises(ContractError):
        features.pack_examples([Ex(1, [FF(3, [1], [1.0])])], 3)
    with pytest.raises(ContractError):
        features.pack_examples([Ex(2, [])], 3)


def test_ragged_batch_round_trip():
    """RaggedBatch (the CSR form K9 unpacks on the device) is lossless against
    the padded layout, including empty fields and empty examples."""
    rng = np.random.default_rng(3)
    n, F, M = 300, 7, 3
    idx = np.full((n, F, M), -1, np.int32)
    val = np.zeros((n, F, M), np.float32)
    cnt = rng.integers(0, M + 1, size=(n, F))
    cnt[::17] = 0
    for e in range(n):
        for f in range(F):
            c = cnt[e, f]
            idx[e, f, :c] = np.sort(rng.choice(1000, c, replace=False))
            val[e, f, :c] = rng.lognormal(size=c)
    rb = features.RaggedBatch.from_padded(idx, val)
    assert rb.ex_off[-1] == (idx >= 0).sum() and rb.cnt.dtype == np.uint8
    assert rb.nbytes() == 8 * (n + 1) + n * F + 8 * int(rb.ex_off[-1])
    i2, v2 = rb.to_padded()
    assert np.array_equal(i2, idx) and np.array_equal(v2, val)


def test_packed_batch_round_trip():
    """PackedBatch (3-byte indices, 1.0 values elided) decodes back to the
    ragged batch bit for bit (host decoder restating K9b)."""
    rng = np.random.default_rng(4)
    n, F, M = 257, 6, 3
    cnt = rng.integers(0, M + 1, size=(n, F))
    idx = np.full((n, F, M), -1, np.int32)
    val = np.zeros((n, F, M), np.float32)
    live = np.arange(M)[None, None, :] < cnt[:, :, None]
    idx[live] = rng.integers(0, 1 << 24, size=int(live.sum()))
    v = np.where(rng.random(int(live.sum())) < 0.3, rng.lognormal(size=int(live.sum())), 1.0)
    v[:5] = [-0.0, 1.0, np.float32(1.0000001), 0.0, 1.0]
    val[live] = v.astype(np.float32)
    rb = features.RaggedBatch.from_padded(idx, val)
    pb = features.PackedBatch.from_ragged(rb)
    assert pb.idx_width == 3 and pb.nbytes() < rb.nbytes()
    nnz = int(rb.ex_off[-1])
    b = pb.idx_bytes.reshape(nnz, 3).astype(np.int64)
    dec_idx = b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16)
    bits = np.unpackbits(pb.vbits, bitorder="little")[:nnz].astype(bool)
    dec_val = np.ones(nnz, np.float32)
    dec_val[bits] = pb.vals
    assert np.array_equal(dec_idx, rb.idx) and np.array_equal(dec_val.view(np.uint32),
                                                              rb.val.view(np.uint32))
    assert np.array_equal(np.cumsum(np.r_[0, bits])[rb.ex_off], pb.voff)


def test_metrics_match_reference():
    g = load("metrics")
    ev = metrics.StreamingEvaluator(30000)
    ev.add_batch(g["scores"][:12345], g["labels"][:12345])
    ev.add_batch(g["scores"][12345:], g["labels"][12345:])
    got = np.array([(i, np.nan if a is None else a) for i, a in ev.auc_series])
    np.testing.assert_allclose(got, g["series"], rtol=1e-12)
    assert ev.mean_logloss == pytest.approx(float(g["mean_logloss"]), rel=1e-12)
    assert metrics.window_auc(g["scores"][:2000], g["labels"][:2000]) == pytest.approx(
        float(g["auc_small"]), rel=1e-12)
    pairs = list(zip(g["scores"][:5000], g["labels"][:5000]))
    assert metrics.logloss(pairs) == pytest.approx(float(g["logloss5k"]), rel=1e-12)
    assert metrics.rig(pairs) == pytest.approx(float(g["rig5k"]), rel=1e-12)
    # SPEC KATs: perfect ranking -> 1.0; all ties -> 0.5; single class -> None
    assert metrics.window_auc([0.1, 0.2, 0.9, 0.8], [0, 0, 1, 1]) == 1.0
    assert metrics.window_auc([0.3] * 6, [0, 1, 0, 1, 1, 0]) == 0.5
    assert metrics.window_auc([0.3, 0.4], [1, 1]) is None


def test_synth_hash_matches_reference_hash_feature():
    g = load("hash")
    got = synth.hash_ranks(torch.as_tensor(g["syn_field"]), torch.as_tensor(g["syn_rank"]), 25)
    assert (got.numpy() == g["syn_bucket"]).all()


def test_synth_examples_are_canonical():
    wl = configs.CFG2
    idx, val = synth.make_examples(wl, 500, seed=3, hash_bits=12)
    assert idx.shape == (500, 24, 3) and idx.dtype == torch.int32
    i = idx.numpy()
    v = val.numpy()
    for e in range(0, 500, 7):
        for f in range(24):
            row = i[e, f]
            live = row[row >= 0]
            assert len(live) >= 1 and (np.diff(live) > 0).all()
            assert (row[len(live):] == -1).all() and (v[e, f, len(live):] == 0).all()
    # categorical fields carry 1.0 (or exact small integers after merging)
    cat = v[:, :20][i[:, :20] >= 0]
    assert set(np.unique(cat)).issubset({1.0, 2.0, 3.0})
    # unsalted variant shares rank->bucket across fields (duplicate stress)
    iu, _ = synth.make_examples(wl, 200, seed=3, hash_bits=12, salted=False)
    assert iu.max() < 4096
