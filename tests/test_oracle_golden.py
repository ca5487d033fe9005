"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/fieldwise_oracle.py) is the checker for every GPU parity
test; these CPU tests are what make it trustworthy.
"""

import math

import numpy as np
import pytest

from oracle import fieldwise_oracle as fo
from tests.golden_io import fixture_flat, load, seeded_flat


# ---------------------------------------------------------------- hashing


def test_fnv_and_hash_feature_match_reference():
    g = load("hash")
    for f, t, b, o in zip(g["fields"], g["tokens"], g["bits"], g["out"]):
        assert fo.hash_feature(str(f), str(t), int(b)) == int(o)
    for raw, o in zip(g["raw"], g["raw_out"]):
        assert fo.fnv1a32(bytes(raw)) == int(o)
    assert fo.fnv1a32(b"a") == 0xE40C292C  # standard FNV-1a vector
    # SPEC S:55-58 KATs
    assert fo.hash_feature("user", "u_42", 18) != fo.hash_feature("ad", "u_42", 18)
    assert fo.hash_feature("x", "anything", 10) < 1024


def test_fnv_batch_matches_scalar():
    g = load("hash")
    items = [str(f).encode() + b"\x1f" + str(t).encode() for f, t in zip(g["fields"], g["tokens"])]
    blob = np.frombuffer(b"".join(items), np.uint8)
    off = np.cumsum([0] + [len(x) for x in items])
    h = fo.fnv1a32_batch(blob, off)
    ref = [fo.fnv1a32(x) for x in items]
    assert (h == np.array(ref, np.uint32)).all()


# ---------------------------------------------------------------- forward


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_oracle_forward_matches_reference(name):
    g = load(f"fwd_{name}")
    F, k, hidden, bits, flat = fixture_flat(g)
    st = fo.OracleStore.from_flat(F, k, hidden, bits, flat)
    idx, val = g["idx"], g["val"]
    for e in range(idx.shape[0]):
        s = fo.forward(fo.row_to_fields(idx[e], val[e]), st)
        assert s["logit"] == pytest.approx(g["logit"][e], rel=1e-12, abs=1e-12)
        assert fo.predict_proba(s["logit"]) == pytest.approx(g["prob"][e], rel=1e-12)
    lg, pb = fo.forward_batch(idx, val, st, chunk=64)
    np.testing.assert_allclose(lg, g["logit"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(pb, g["prob"], rtol=1e-10)


def test_forward_spec_kats():
    # 2 fields, k=1, w_{a,f2}=0.5, w_{b,f1}=0.25 -> pair output 0.125
    st = fo.OracleStore.zeros(2, 1, (), 4)
    st.ffm[3, 1, 0] = 0.5  # feature a=3 in field 0, toward field 1
    st.ffm[5, 0, 0] = 0.25  # feature b=5 in field 1, toward field 0
    fields = [(0, np.array([3]), np.array([1.0])), (1, np.array([5]), np.array([1.0]))]
    s = fo.forward(fields, st)
    assert s["pairs"][0] == 0.125
    assert s["logit"] == 0.125  # S:127 no hidden layers -> lr + sum(pairs)
    # S:126 empty example -> logit = bias
    st.lr[st.n_features] = 0.75
    assert fo.forward([], st)["logit"] == 0.75
    # S:131-134
    assert fo.predict_proba(0.0) == 0.5
    assert fo.predict_proba(2.0) == pytest.approx(0.8807970779778823, rel=1e-15)
    assert fo.predict_proba(-2.0) == pytest.approx(1 - 0.8807970779778823, rel=1e-14)
    # S:156 pair count
    assert len(fo.pair_indices(24)[0]) == 276


# ---------------------------------------------------------------- training


@pytest.mark.parametrize("name", ["salted", "unsalted", "pt025_dense", "ffm_lr"])
def test_oracle_training_matches_reference(name):
    g = load(f"train_{name}")
    F, k, bits = int(g["F"]), int(g["k"]), int(g["bits"])
    hidden = tuple(int(h) for h in g["hidden"])
    flat = seeded_flat(F, k, hidden, bits, g["w_seed"], 0.05)
    assert float(flat.astype(np.float64).sum()) == float(g["init_sum"])
    st = fo.OracleStore.from_flat(F, k, hidden, bits, flat)
    lr, pt = float(g["lr"]), float(g["power_t"])
    probs, _ = fo.train_sequential(g["idx"], g["val"], g["labels"], st, lr, lr, lr, pt,
                                   sparse=bool(g["sparse"]))
    np.testing.assert_allclose(probs, g["probs"], rtol=1e-12, atol=0)
    final = st.flat(True)
    ref = g["final"]
    # the oracle restates the reference op for op: expect (near) bit-identity
    mism = np.flatnonzero(final.view(np.uint32) != ref.view(np.uint32))
    assert len(mism) <= 2, f"{len(mism)} slots differ"
    np.testing.assert_allclose(final, ref, rtol=1e-6, atol=1e-9)


def test_adagrad_scalar_kat():
    # single lr weight, x=1, acc0=1, power_t=0.5 -> hand-computed step
    st = fo.OracleStore.zeros(1, 1, (), 4)
    fields = [(0, np.array([2]), np.array([1.0]))]
    s = fo.forward(fields, st)
    fo.backward_update(s, fields, 1, st, 0.1, 0.1, 0.1, 0.5)
    g = 0.5 - 1.0
    acc = 1.0 + g * g
    assert st.lr_acc[2] == np.float32(acc)
    assert st.lr[2] == np.float32(0.0 - 0.1 * g * (1.0 / math.sqrt(acc)))


def test_sparse_equals_dense_bytes():
    g = load("train_unsalted")
    F, k, bits = int(g["F"]), int(g["k"]), int(g["bits"])
    hidden = tuple(int(h) for h in g["hidden"])
    flat = seeded_flat(F, k, hidden, bits, g["w_seed"], 0.05)
    a = fo.OracleStore.from_flat(F, k, hidden, bits, flat)
    b = a.copy()
    n = 60
    fo.train_sequential(g["idx"][:n], g["val"][:n], g["labels"][:n], a, .1, .1, .1, .5, True)
    fo.train_sequential(g["idx"][:n], g["val"][:n], g["labels"][:n], b, .1, .1, .1, .5, False)
    assert a.flat().tobytes() == b.flat().tobytes()


# ---------------------------------------------------------------- context cache


def test_context_cache_matches_merged_forward():
    g = load("ctx")
    F, k, hidden, bits, flat = fixture_flat(g)
    st = fo.OracleStore.from_flat(F, k, hidden, bits, flat)
    R, C = g["prob"].shape
    for r in range(R):
        cache = fo.build_context_cache(fo.row_to_fields(g["ctx_idx"][r], g["ctx_val"][r]), st)
        for c in range(C):
            cf = [(f + int(g["Fc"]), i, v) for f, i, v in
                  fo.row_to_fields(g["cand_idx"][r, c], g["cand_val"][r, c])]
            _, p = fo.predict_with_cache(cache, cf, st)
            assert abs(p - g["prob"][r, c]) <= 1e-12  # S:266 asks 1e-6


def test_context_cache_opcount_reduction():
    # S:270 / S:524: 100 candidates sharing a 20-field context -> >= 3x fewer FFM madds
    F, Fc = 24, 20
    st = fo.random_store(F, 4, (), 10, seed=3)
    rng = np.random.default_rng(0)
    ctx = [(f, np.array([int(rng.integers(1024))]), np.array([1.0])) for f in range(Fc)]
    cands = [[(f, np.array([int(rng.integers(1024))]), np.array([1.0])) for f in range(Fc, F)]
             for _ in range(100)]
    cached = [0]
    cache = fo.build_context_cache(ctx, st, cached)
    probs_c = [fo.predict_with_cache(cache, c, st, cached)[1] for c in cands]
    uncached = [0]
    probs_u = [fo.predict_proba(fo.forward(ctx + c, st, uncached)["logit"]) for c in cands]
    np.testing.assert_allclose(probs_c, probs_u, atol=1e-12)
    assert uncached[0] >= 3 * cached[0]


# ---------------------------------------------------------------- quantisation


def test_quant_spec_kats():
    # W={0,1}, alpha=beta=4 -> bucket 1/65536; 0.5 -> 32768; max -> 65535
    hmin, hb, q = fo.quantize(np.array([0.0, 1.0, 0.5], np.float32))
    assert hmin == 0.0 and hb == np.float32(1.0 / 65536)
    assert q.tolist() == [0, 65535, 32768]
    # constant W with <= alpha decimals -> bucket 0, all indices 0
    hmin, hb, q = fo.quantize(np.full(10, 0.25, np.float32))
    assert hb == 0.0 and (q == 0).all() and hmin == np.float32(0.25)
    # index 0 dequantises to exactly w_min; S:328 bucket 0 -> constant
    assert fo.dequantize(np.float32(-0.3), np.float32(1e-5), np.array([0], np.uint16))[0] \
        == np.float32(-0.3)
    assert (fo.dequantize(np.float32(0.25), np.float32(0), np.zeros(5, np.uint16)) == 0.25).all()


def test_quant_roundtrip_bound_and_monotone():
    rng = np.random.default_rng(1)
    w = (rng.standard_normal(200_000) * 0.05).astype(np.float32)
    hmin, hb, q = fo.quantize(w)
    back = fo.dequantize(hmin, hb, q)
    err = np.abs(back.astype(np.float64) - w)
    inner = (q > 0) & (q < 65535)
    # S:365 bound + the f32 rounding slack the header and the f32 mul/add add
    slack = 65536 * np.spacing(hb) + 2 * np.spacing(np.float32(np.abs(w).max()))
    assert err[inner].max() <= hb / 2 + slack
    order = np.argsort(w, kind="stable")
    assert (np.diff(q[order].astype(np.int64)) >= 0).all()


# ------------------------------------------------------------------ transfer


def test_oracle_varint_and_patch_spec_examples():
    assert fo.encode_varint(0) == b"\x00"
    assert fo.encode_varint(127) == b"\x7f"
    assert fo.encode_varint(128) == b"\x80\x01"
    rng = np.random.default_rng(0)
    for v in rng.integers(0, 2**63, 2000).tolist() + [2**64 - 1]:
        e = fo.encode_varint(v)
        assert fo.decode_varint(e) == (v, len(e))
    p = fo.create_patch(bytes([1, 2, 3, 4]), bytes([1, 2, 9, 4]))
    assert p[32:] == bytes([2, 1, 9])
    assert fo.apply_patch(bytes([1, 2, 3, 4]), p) == bytes([1, 2, 9, 4])
    assert len(fo.create_patch(b"xyz", b"xyz")) == 32
    # gap rule: runs 3 identical bytes apart merge, 4 apart do not
    assert fo.diff_ops(b"aaaaaaaaaa", b"Xaaa" + b"Xaaaaa") == [(0, 5)]
    assert fo.diff_ops(b"aaaaaaaaaa", b"Xaaaa" + b"Xaaaa") == [(0, 1), (5, 6)]


def test_host_digest_and_varints_match_oracle():
    from paper_2407_10115_b200 import transfer
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 1000):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert transfer.digest(b) == fo.fnv1a64(b)
    for v in (0, 1, 127, 128, 300, 2**35 + 7, 2**64 - 1):
        assert transfer.encode_varint(v) == fo.encode_varint(v)
        assert transfer.decode_varint(transfer.encode_varint(v)) == (v, len(fo.encode_varint(v)))
