"""The reference's public per-example API and text-source loops, on the GPU,
against golden outputs of the reference itself (tests/golden/api.npz, made by
tests/golden/make_golden.py importing /root/reference):

* ForwardState intermediates (M:275-290) from model.forward (K11 trace)
* mac_counter (M:130-139) and loss_gradients (M:575-634)
* the literal T:175-185 loop: forward -> predict_proba -> backward_update
* train_stream / hogwild_train(n_threads=1) / evaluate_stream over text lines
  with blank and unparseable lines (T:172-236)

Bar: predictions / intermediates within 1e-5 relative (f64 here: 1e-9 with an
absolute floor), weights |dw| <= 1e-5 max(|w|, 1e-3)."""

import numpy as np
import pytest
import torch

from paper_2407_10115_b200 import model as pm
from paper_2407_10115_b200 import training as pt
from paper_2407_10115_b200.errors import ContractError, NumericError, TrainAborted
from paper_2407_10115_b200.features import (InputSchema, ParsedExample, parse_example,
                                            serialize_example)
from paper_2407_10115_b200.model import ModelConfig, WeightStore
from tests.golden_io import load, seeded_flat

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _setup():
    g = load("api")
    F, k, bits = int(g["F"]), int(g["k"]), int(g["bits"])
    hidden = tuple(int(h) for h in g["hidden"])
    cfg = ModelConfig(n_fields=F, k=k, hidden_sizes=hidden, hash_bits=bits, lr_ffm=0.1,
                      lr_lr=0.1, lr_nn=0.1, power_t=0.5)
    flat = seeded_flat(F, k, hidden, bits, g["w_seed"], g["scale"])
    store = WeightStore.from_flat(cfg, flat, DEV)  # accumulators 1.0 (M:682-683)
    schema = InputSchema(tuple(str(x) for x in g["names"]), frozenset(), bits)
    return g, cfg, store, schema


def _example(g, schema, e):
    from paper_2407_10115_b200.features import FieldFeatures
    idx, val = g["idx"][e], g["val"][e]
    fields = []
    for f in range(idx.shape[0]):
        sel = idx[f] >= 0
        if sel.any():
            fields.append(FieldFeatures(f, idx[f][sel].astype(np.int64),
                                        val[f][sel].astype(np.float64)))
    return ParsedExample(int(g["labels"][e]), tuple(fields))


def close(a, b, rel=1e-9, floor=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), floor / rel))


def close_weights(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return int((np.abs(got - ref) > 1e-5 * np.maximum(np.abs(ref), 1e-3)).sum())


def test_forward_state_intermediates_match_reference():
    g, cfg, store, schema = _setup()
    for e in range(8):
        ex = _example(g, schema, e)
        mc = pm.OpCounter()
        s = pm.forward(ex, store, mac_counter=mc)
        assert close(s.lr_out, g[f"e{e}_lr_out"])
        assert close(s.logit, g[f"e{e}_logit"])
        assert close(s.ffm_pair_outputs, g[f"e{e}_pairs"])
        assert close(s.latent_sums, g[f"e{e}_S"])
        assert close(s.merge_vec, g[f"e{e}_v"])
        assert close([s.merge_mu, s.merge_sd], g[f"e{e}_mu_sd"])
        assert close(s.merged_input, g[f"e{e}_merged"], rel=1e-7, floor=1e-9)
        for li in range(len(cfg.hidden_sizes)):
            assert close(s.layer_pre_acts[li], g[f"e{e}_pre{li}"], rel=1e-7, floor=1e-9)
            assert close(s.layer_acts[li], g[f"e{e}_act{li}"], rel=1e-7, floor=1e-9)
        assert mc.madds == int(g[f"e{e}_macs"])
        assert s._store is store and s._store_version == store.version


def test_loss_gradients_match_reference():
    g, cfg, store, schema = _setup()
    for e in range(8):
        ex = _example(g, schema, e)
        s = pm.forward(ex, store)
        grad = pm.loss_gradients(s, ex, int(g["labels"][e]), store)
        ref = g[f"e{e}_grad"]
        assert grad.shape == ref.shape == (store.weights_total,)
        scale = np.abs(ref).max()
        assert np.abs(grad - ref).max() <= 1e-9 * scale
        assert np.array_equal(grad == 0, ref == 0)  # same sparsity (untouched rows)


def test_reference_loop_forward_predict_backward():
    """T:175-185 literally, per ParsedExample, against the reference's loop."""
    g, cfg, store, schema = _setup()
    n = g["idx"].shape[0]
    ps, losses = [], []
    for e in range(n):
        ex = _example(g, schema, e)
        s = pm.forward(ex, store)
        ps.append(pm.predict_proba(s.logit))
        losses.append(pm.backward_update(s, ex, ex.label, store))
    assert np.max(np.abs(np.array(ps) - g["loop_p"]) / g["loop_p"]) < 1e-5
    assert np.max(np.abs(np.array(losses) - g["loop_loss"]) / g["loop_loss"]) < 1e-5
    assert close_weights(store.weight_values(True), g["loop_final"]) == 0
    assert store.version == int(g["loop_version"])


def test_backward_update_contracts():
    g, cfg, store, schema = _setup()
    ex = _example(g, schema, 3)
    s = pm.forward(ex, store)
    with pytest.raises(ContractError):
        pm.backward_update(s, ex, 2, store)
    pm.backward_update(s, ex, 1, store)
    with pytest.raises(ContractError):  # stale state: the store moved on (M:451-452)
        pm.backward_update(s, ex, 1, store)
    with pytest.raises(ContractError):
        pm.loss_gradients(s, ex, 1, store)


def test_forward_nonfinite_diagnosis_block():
    g, cfg, store, schema = _setup()
    ex = _example(g, schema, 5)
    store.lr[store.n_features] = float("inf")  # bias -> lr block (M:308-318)
    with pytest.raises(NumericError) as ei:
        pm.forward(ex, store)
    assert ei.value.block == "lr"


def test_train_stream_text_matches_reference():
    g, cfg, store, schema = _setup()
    text = str(g["text"]).splitlines(keepends=True)
    rep = pt.train_stream(iter(text), store, schema)
    assert rep.examples_seen == int(g["ts_seen"])
    assert rep.parse_errors == int(g["ts_parse_errors"])
    assert rep.progressive_logloss == pytest.approx(float(g["ts_logloss"]), rel=1e-6)
    ser = np.array([(i, np.nan if a is None else a) for i, a in rep.rolling_auc_series])
    assert ser.shape == g["ts_series"].shape
    assert close_weights(store.weight_values(True), g["ts_final"]) == 0
    assert store.version == int(g["ts_version"])


def test_hogwild_one_worker_text_matches_reference():
    g, cfg, store, schema = _setup()
    text = str(g["text"]).splitlines(keepends=True)
    v0 = store.version
    rep = pt.hogwild_train(iter(text), store, schema, pt.TrainOptions(n_threads=1))
    assert rep.examples_seen == int(g["hw_seen"])
    assert rep.parse_errors == int(g["hw_parse_errors"])
    assert rep.progressive_logloss == pytest.approx(float(g["hw_logloss"]), rel=1e-6)
    assert close_weights(store.weight_values(True), g["hw_final"]) == 0
    assert store.version == v0 + 1  # mark_mutated once (T:318)


def test_evaluate_stream_text_matches_reference():
    g, cfg, store, schema = _setup()
    store.load_flat(g["ts_final"])
    text = [t for t in str(g["text"]).splitlines(keepends=True)
            if not t.startswith("2 ") and ("|" in t or not t.strip())]
    auc, ll, n = pt.evaluate_stream(iter(text), store, schema)
    assert n == int(g["ev_n"])
    assert auc == pytest.approx(float(g["ev_auc"]), abs=1e-6)  # K1 probs are f32
    assert ll == pytest.approx(float(g["ev_logloss"]), rel=1e-6)
    from paper_2407_10115_b200.errors import ParseError
    with pytest.raises(ParseError):
        pt.evaluate_stream(iter(text[:3] + ["2 |c0 @1\n"]), store, schema)
    auc0, ll0, n0 = pt.evaluate_stream(iter(["  \n"]), store, schema)
    assert auc0 is None and np.isnan(ll0) and n0 == 0


def test_train_stream_source_failure_attaches_partial_report():
    g, cfg, store, schema = _setup()
    text = str(g["text"]).splitlines(keepends=True)

    def source():
        yield from text[:50]
        raise TrainAborted("I/O failure reading chunk 2")

    with pytest.raises(TrainAborted) as ei:
        pt.train_stream(source(), store, schema)
    rep = ei.value.partial_report
    assert rep is not None and 0 < rep.examples_seen <= 50


def test_parse_example_and_serialize_round_trip():
    g, cfg, store, schema = _setup()
    for e in range(2, 30):
        ex = _example(g, schema, e)
        line = serialize_example(ex, schema)
        back = parse_example(line, schema)
        assert back.label == ex.label and len(back.fields) == len(ex.fields)
        for a, b in zip(back.fields, ex.fields):  # K10 values: exact or within 4 f64 ulp
            assert a.field_id == b.field_id and np.array_equal(a.indices, b.indices)
            assert np.allclose(a.values, b.values, rtol=1e-15, atol=0)


def test_hashing_api_matches_reference_vectors():
    from paper_2407_10115_b200 import hashing as ph
    h = load("hash")
    for f, t, b, o in list(zip(h["fields"], h["tokens"], h["bits"], h["out"]))[:40]:
        assert ph.hash_feature(str(f), str(t), int(b)) == int(o)
    for raw, o in zip(h["raw"], h["raw_out"]):
        assert ph.fnv1a32(bytes(raw)) == int(o)
    assert ph.fnv1a64(b"") == 0xCBF29CE484222325
    assert ph.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
