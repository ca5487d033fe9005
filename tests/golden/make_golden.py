"""Generate the golden fixtures by running the REFERENCE itself.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture stores the inputs (so no test regenerates them) and the
outputs of the unmodified reference package ``fieldwise``:

* ``hash.npz``      -- fnv1a32 / hash_feature vectors (H:28-50) and the
                       synthetic rank->bucket map checked against H:43
* ``fwd_*.npz``     -- model.forward + predict_proba (M:300-397) over seeded
                       padded examples against a seeded flat store
* ``train_*.npz``   -- training.train_stream (T:188-218) over the same kind
                       of examples: per-example progressive probabilities and
                       the final flat store bytes (weights + accumulators)
* ``ctx.npz``       -- forward on merged context+candidate examples (the
                       truth SPEC S:266 names for the context cache)
* ``metrics.npz``   -- StreamingEvaluator / window_auc / logloss (Me:21-129)
* ``serial.npz``    -- flat_weight_view bytes (M:640-660)
* ``parse.npz``     -- features.parse_example (Fe:175-235) over seeded text
                       lines with edge cases: which lines raise ParseError,
                       labels, canonical (field, index, value) per line
* ``api.npz``       -- the per-example API and the text-source loops:
                       ForwardState intermediates (M:275-290), mac_counter
                       (M:130-139), loss_gradients (M:575-634), the literal
                       T:175-185 loop, train_stream / hogwild_train(1) /
                       evaluate_stream (T:188-236) over text lines with blank
                       and unparseable lines

Nothing here runs on the GPU box; /root/reference does not exist there.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from fieldwise import hashing as rh  # noqa: E402
from fieldwise import metrics as rmet  # noqa: E402
from fieldwise import model as rm  # noqa: E402
from fieldwise import training as rt  # noqa: E402
from fieldwise.features import FieldFeatures, InputSchema, ParsedExample, serialize_example  # noqa: E402

from paper_2407_10115_b200 import configs, synth  # noqa: E402


def ref_store(F, k, hidden, bits, flat_w):
    """Reference WeightStore holding ``flat_w`` weights and acc = 1.0."""
    cfg = rm.ModelConfig(n_fields=F, k=k, hidden_sizes=tuple(hidden), hash_bits=bits,
                         lr_ffm=0.1, lr_lr=0.1, lr_nn=0.1, power_t=0.5)
    st = rm.WeightStore(cfg)
    st.flat[: st.weights_total] = flat_w
    st.flat[st.acc_offset:] = 1.0
    return st


def sha(a):
    import hashlib
    return np.array(hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest())


def seeded_flat(F, k, hidden, bits, seed, scale):
    cfg = rm.ModelConfig(n_fields=F, k=k, hidden_sizes=tuple(hidden), hash_bits=bits)
    n = rm.WeightStore(cfg).weights_total
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n) * scale).astype(np.float32)


def to_example(idx_row, val_row, label=0):
    fields = []
    for f in range(idx_row.shape[0]):
        sel = idx_row[f] >= 0
        if not sel.any():
            continue
        fields.append(FieldFeatures(f, idx_row[f][sel].astype(np.int64),
                                    val_row[f][sel].astype(np.float64)))
    return ParsedExample(int(label), tuple(fields))


def gen_inputs(wl, n, bits, seed, salted=True):
    idx, val = synth.make_examples(wl, n, seed=seed, hash_bits=bits, salted=salted)
    return idx.numpy(), val.numpy()


def fwd_fixture(name, wl, n, bits, seed, scale, bf16=False, extra_edge=True):
    F, k, hidden = wl.n_fields, wl.k, wl.hidden
    idx, val = gen_inputs(wl, n, bits, seed)
    if extra_edge:
        # edge rows: an all-empty example, a single-field example, a row with
        # only numeric fields, a duplicate-bucket-across-fields row
        idx[0] = -1
        val[0] = 0
        idx[1, 1:] = -1
        val[1, 1:] = 0
        idx[2, : F // 2] = -1
        val[2, : F // 2] = 0
        idx[3, :, 0] = 7
        idx[3, :, 1:] = -1
        val[3, :, 1:] = 0
    flat = seeded_flat(F, k, hidden, bits, seed + 17, scale)
    if bf16:
        import torch
        flat = torch.from_numpy(flat).to(torch.bfloat16).to(torch.float32).numpy()
    st = ref_store(F, k, hidden, bits, flat)
    logit = np.empty(n)
    prob = np.empty(n)
    lr_out = np.empty(n)
    pairsum = np.empty(n)
    for e in range(n):
        s = rm.forward(to_example(idx[e], val[e]), st)
        logit[e] = s.logit
        prob[e] = rm.predict_proba(s.logit)
        lr_out[e] = s.lr_out
        pairsum[e] = float(s.ffm_pair_outputs.sum())
    np.savez_compressed(os.path.join(HERE, f"fwd_{name}.npz"), idx=idx, val=val,
                        w_seed=seed + 17, scale=scale, bf16=bf16, flat_sha=sha(flat),
                        F=F, k=k, hidden=np.array(hidden, np.int64), bits=bits,
                        logit=logit, prob=prob, lr_out=lr_out, pairsum=pairsum)
    print("fwd", name, n, "examples")


def train_fixture(name, wl, n, bits, seed, salted, power_t=0.5, sparse=True, lr=0.1):
    F, k, hidden = wl.n_fields, wl.k, wl.hidden
    idx, val = gen_inputs(wl, n, bits, seed, salted=salted)
    rng = np.random.default_rng(seed + 5)
    labels = (rng.random(n) < 0.35).astype(np.uint8)
    flat_w = seeded_flat(F, k, hidden, bits, seed + 17, 0.05)
    cfg = rm.ModelConfig(n_fields=F, k=k, hidden_sizes=tuple(hidden), hash_bits=bits,
                         lr_ffm=lr, lr_lr=lr, lr_nn=lr, power_t=power_t)
    st = rm.WeightStore(cfg)
    st.flat[: st.weights_total] = flat_w
    st.flat[st.acc_offset:] = 1.0
    names = tuple(f"f{f}" for f in range(F))
    schema = InputSchema(names, frozenset(), max(bits, 10))
    lines = [serialize_example(to_example(idx[e], val[e], labels[e]), schema) for e in range(n)]
    # progressive probabilities, recorded through the reference loop itself
    probs = []
    class Rec(rmet.StreamingEvaluator):
        def add(self, score, label):
            probs.append(score)
            super().add(score, label)

    saved = rt.StreamingEvaluator
    rt.StreamingEvaluator = Rec
    try:
        rep = rt.train_stream(iter(lines), st, schema, rt.TrainOptions(sparse_updates=sparse))
    finally:
        rt.StreamingEvaluator = saved
    assert rep.examples_seen == n, rep.summary()
    np.savez_compressed(os.path.join(HERE, f"train_{name}.npz"), idx=idx, val=val,
                        labels=labels, F=F, k=k, hidden=np.array(hidden, np.int64), bits=bits,
                        w_seed=seed + 17, init_sum=np.float64(flat_w.astype(np.float64).sum()),
                        lr=lr, power_t=power_t, sparse=sparse,
                        probs=np.array(probs), logloss=rep.progressive_logloss,
                        final=st.flat.copy())
    print("train", name, n, "examples; logloss", rep.progressive_logloss)


def hash_fixture():
    rng = np.random.default_rng(7)
    fields, tokens, bits, out = [], [], [], []
    for i in range(400):
        f = "".join(chr(97 + c) for c in rng.integers(0, 26, rng.integers(0, 6)))
        t = "".join(chr(33 + c) for c in rng.integers(0, 90, rng.integers(0, 12)))
        b = int(rng.integers(10, 30))
        fields.append(f)
        tokens.append(t)
        bits.append(b)
        out.append(rh.hash_feature(f, t, b))
    fields += ["user", "ad", "ünï", ""]
    tokens += ["u_42", "u_42", "tøk€n", ""]
    bits += [18, 18, 20, 10]
    out += [rh.hash_feature(f, t, b) for f, t, b in zip(fields[-4:], tokens[-4:], bits[-4:])]
    raw = [b"", b"a", b"foobar", b"\x00\xff" * 9, bytes(range(256))]
    raw_out = [rh.fnv1a32(x) for x in raw]
    # synthetic rank->bucket map: hash_feature(f"f{field}", f"t{r}", b)
    fr = rng.integers(0, 40, 3000)
    rr = rng.integers(1, 1 << 25, 3000)
    rr[:10] = [1, 9, 10, 99, 100, 12345678, 33554432, 2, 5, 1000000]
    syn = np.array([rh.hash_feature(f"f{f}", f"t{r}", 25) for f, r in zip(fr, rr)], np.int64)
    np.savez_compressed(os.path.join(HERE, "hash.npz"),
                        fields=np.array(fields, dtype=object), tokens=np.array(tokens, dtype=object),
                        bits=np.array(bits), out=np.array(out, np.int64),
                        raw=np.array(raw, dtype=object), raw_out=np.array(raw_out, np.int64),
                        syn_field=fr, syn_rank=rr, syn_bucket=syn, allow_pickle=True)
    print("hash", len(out))


def ctx_fixture():
    wl = configs.CFG4
    F, k, hidden, bits = wl.n_fields, wl.k, wl.hidden, 12
    R, C, Fc = 6, 40, wl.ctx_fields
    ctx_idx, ctx_val = synth.make_examples(wl, R, seed=91, hash_bits=bits, n_fields=Fc)
    cand_idx, cand_val = synth.make_examples(wl, R * C, seed=92, hash_bits=bits,
                                             field_offset=Fc, n_fields=F - Fc)
    ctx_idx, ctx_val = ctx_idx.numpy(), ctx_val.numpy()
    cand_idx = cand_idx.numpy().reshape(R, C, F - Fc, 1)
    cand_val = cand_val.numpy().reshape(R, C, F - Fc, 1)
    # edge cases: empty context (request 0), empty candidate (r1,c0), partial
    ctx_idx[0] = -1
    ctx_val[0] = 0
    cand_idx[1, 0] = -1
    cand_val[1, 0] = 0
    cand_idx[2, 1, :4] = -1
    cand_val[2, 1, :4] = 0
    flat = seeded_flat(F, k, hidden, bits, 93, 0.05)
    st = ref_store(F, k, hidden, bits, flat)
    prob = np.empty((R, C))
    for r in range(R):
        for c in range(C):
            merged = np.concatenate([ctx_idx[r], cand_idx[r, c]], axis=0)
            mval = np.concatenate([ctx_val[r], cand_val[r, c]], axis=0)
            prob[r, c] = rm.predict_proba(rm.forward(to_example(merged, mval), st).logit)
    np.savez_compressed(os.path.join(HERE, "ctx.npz"), ctx_idx=ctx_idx, ctx_val=ctx_val,
                        cand_idx=cand_idx, cand_val=cand_val, w_seed=93, scale=0.05,
                        flat_sha=sha(flat), F=F, k=k,
                        hidden=np.array(hidden, np.int64), bits=bits, Fc=Fc, prob=prob)
    print("ctx", R, C)


def metrics_fixture():
    rng = np.random.default_rng(11)
    n = 70000
    labels = (rng.random(n) < 0.3).astype(np.int64)
    scores = np.clip(0.3 + 0.2 * (labels - 0.3) + 0.2 * rng.standard_normal(n), 0, 1)
    scores[:500] = 0.5  # ties
    ev = rmet.StreamingEvaluator(30000)
    for s, y in zip(scores, labels):
        ev.add(float(s), int(y))
    auc_small = rmet.window_auc(scores[:2000], labels[:2000])
    ll = rmet.logloss(zip(scores[:5000], labels[:5000]))
    rg = rmet.rig(list(zip(scores[:5000], labels[:5000])))
    series = np.array([(i, np.nan if a is None else a) for i, a in ev.auc_series])
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), labels=labels, scores=scores,
                        series=series, mean_logloss=ev.mean_logloss, auc_small=auc_small,
                        logloss5k=ll, rig5k=rg)
    print("metrics", series.shape)


def serial_fixture():
    cfg = rm.ModelConfig(n_fields=3, k=2, hidden_sizes=(4,), hash_bits=4, init_seed=5)
    st = rm.init_model(cfg)
    full = rm.flat_weight_view(st, True)
    infer = rm.flat_weight_view(st, False)
    np.savez_compressed(os.path.join(HERE, "serial.npz"),
                        full=np.frombuffer(full, np.uint8), infer=np.frombuffer(infer, np.uint8),
                        cfg_json=np.array(cfg.to_json()))
    print("serial", len(full), len(infer))


def _value_text(rng):
    r = rng.random()
    if r < 0.25:
        return str(int(rng.integers(-5, 100)))
    if r < 0.45:
        return f"{rng.random() * 10:.{int(rng.integers(1, 6))}f}"
    if r < 0.6:
        return repr(float(rng.standard_normal() * 10 ** int(rng.integers(-8, 9))))
    if r < 0.7:
        return f"{rng.integers(1, 999)}e{int(rng.integers(-30, 30))}"
    if r < 0.75:
        return "1_000.2_5"
    if r < 0.8:
        return f"+.{rng.integers(0, 99999)}"
    if r < 0.85:
        return f"{rng.integers(0, 9)}."
    if r < 0.9:
        return f"{rng.integers(1, 9)}E+0{rng.integers(0, 9)}"
    return repr(float(rng.lognormal()))


def parse_fixture():
    from fieldwise.errors import ParseError
    from fieldwise.features import parse_example
    rng = np.random.default_rng(11)
    names = ["user", "ad", "site", "hour", "price", "cnt", "q", "dev", "os", "geo"]
    schema = InputSchema(tuple(names), frozenset({"price", "cnt"}), 20)
    ws = [" ", "  ", "\t", " \t ", "\x1f", " \x0b"]
    words = ["a", "b1", "u_42", "x.y", "tok-9", "Z", "ünï", "€", "@", "@12a", "@7", "@0042",
             "@1048575", "@99", "-", "a:b"]
    lines = []
    for i in range(700):
        label = ["0", "1", "-1", " 1 ", "1\t", " 0"][int(rng.integers(0, 6))]
        parts = [label]
        for _ in range(int(rng.integers(1, 7))):
            f = names[int(rng.integers(0, len(names)))]
            toks = []
            for _ in range(int(rng.integers(0, 8))):
                w = words[int(rng.integers(0, len(words)))] if rng.random() < 0.4 else \
                    f"t{int(rng.integers(0, 40))}"
                if rng.random() < 0.35:
                    w = w + ":" + _value_text(rng)
                toks.append(w)
            sep = ws[int(rng.integers(0, len(ws)))]
            parts.append("|" + f + (sep if toks else "") + sep.join(toks) +
                         (sep if rng.random() < 0.2 else ""))
        lines.append("".join(parts) if rng.random() < 0.5 else " ".join(parts))
    lines += [  # errors and edges (Fe:191-231)
        "2 |user a", "|user a", "1", "1 |", "1 | ", "1 |user a |", "1 |zzz a", "1 |user a:abc",
        "1 |user a:inf", "1 |user a:nan", "1 |user a:-Infinity", "1 |user @1048576",
        "1 |user @99999999999999999999", "1 |user a:1__0", "1 |user a:_1", "1 |user a:1_",
        "1 |user a:1e", "1 |user a:e5", "1 |user a:.", "1 |user a:", "1 |user a:0x10",
        "1 |user a:1e400", "1 |user a:1e-400", "1 |user a:-0.0", "1 |user a:1e1_0",
        "1 |user a:1._5", "1 |user a:+-1", "0 |price 3:2.5 3:0.5 x:-1 @5:4", "1 |cnt a a a:2",
        "-1 |user a |user a |ad a", "1 |user a:1:2", "1 |user\ta\x1fb\x1cc", "", "   ",
        "1 |user " + " ".join(f"t{j}" for j in range(250)),
        "1 |q " + " ".join(f"w:{j * 0.37:.3f}" for j in range(60)) + " |q w:1",
        "1 |price 0.0000000000000000000000012345678901234567890123 1e-310:1 big:" + "9" * 30,
        "1 |user 123456789012345678901234567890:1.7976931348623157e308",
        "1 |user a:4.9e-324 b:2.2250738585072014e-308 c:0.1 d:0.3 e:12345678901234567e-10",
    ]
    ok, labels, off, fid, idx, val = [], [], [0], [], [], []
    for ln in lines:
        try:
            ex = parse_example(ln, schema)
        except ParseError:
            ok.append(False)
            labels.append(0)
            off.append(off[-1])
            continue
        ok.append(True)
        labels.append(ex.label)
        for ff in sorted(ex.fields, key=lambda f: f.field_id):
            fid += [ff.field_id] * len(ff.indices)
            idx += ff.indices.tolist()
            val += ff.values.tolist()
        off.append(len(idx))
    text = "\n".join(lines) + "\n"
    np.savez_compressed(os.path.join(HERE, "parse.npz"),
                        text=np.frombuffer(text.encode("utf-8"), np.uint8),
                        schema=np.array(schema.to_text()), ok=np.array(ok),
                        labels=np.array(labels, np.uint8), ex_off=np.array(off, np.int64),
                        fid=np.array(fid, np.int64), idx=np.array(idx, np.int64),
                        val=np.array(val, np.float64))
    print("parse", len(lines), "lines,", sum(ok), "ok,", len(idx), "features")


def api_fixture():
    """Reference outputs of the per-example API and the text-source loops."""
    wl = configs.CFG3
    F, k, hidden, bits = 6, 4, (16, 8), 10
    n = 240
    idx, val = synth.make_examples(wl, n, seed=131, hash_bits=bits, salted=False,
                                   n_fields=F)
    idx, val = idx.numpy(), val.numpy()
    idx[0] = -1  # all-empty example
    val[0] = 0
    idx[1, 1:] = -1  # single field
    val[1, 1:] = 0
    rng = np.random.default_rng(132)
    labels = (rng.random(n) < 0.4).astype(np.uint8)
    flat = seeded_flat(F, k, hidden, bits, 133, 0.1)
    names = tuple(f"c{f}" for f in range(F))
    schema = InputSchema(names, frozenset(), bits)
    lines = [serialize_example(to_example(idx[e], val[e], labels[e]), schema) for e in range(n)]
    # text stream with blank and unparseable lines sprinkled in (T:176-181)
    text = []
    for e, ln in enumerate(lines):
        if e % 37 == 5:
            text.append("   \n")
        if e % 53 == 7:
            text.append("2 |c0 @1\n")  # bad label: counted, skipped
        text.append(ln + "\n")
    # ForwardState / mac_counter / loss_gradients on the first 8 examples
    st = ref_store(F, k, hidden, bits, flat)
    keep = {}
    for e in range(8):
        ex = to_example(idx[e], val[e], labels[e])
        mc = rm.OpCounter()
        s = rm.forward(ex, st, mac_counter=mc)
        keep[f"e{e}_lr_out"] = s.lr_out
        keep[f"e{e}_logit"] = s.logit
        keep[f"e{e}_pairs"] = s.ffm_pair_outputs
        keep[f"e{e}_merged"] = s.merged_input
        keep[f"e{e}_S"] = s.latent_sums
        keep[f"e{e}_v"] = s.merge_vec
        keep[f"e{e}_mu_sd"] = np.array([s.merge_mu, s.merge_sd])
        for li, (z, a) in enumerate(zip(s.layer_pre_acts, s.layer_acts)):
            keep[f"e{e}_pre{li}"] = z
            keep[f"e{e}_act{li}"] = a
        keep[f"e{e}_macs"] = mc.madds
        keep[f"e{e}_grad"] = rm.loss_gradients(s, ex, int(labels[e]), st)
    # the literal T:175-185 loop: forward -> predict_proba -> backward_update
    st = ref_store(F, k, hidden, bits, flat)
    loop_p, loop_loss = [], []
    for e in range(n):
        ex = to_example(idx[e], val[e], labels[e])
        s = rm.forward(ex, st)
        loop_p.append(rm.predict_proba(s.logit))
        loop_loss.append(rm.backward_update(s, ex, ex.label, st))
    loop_final = st.flat.copy()
    loop_version = st.version
    # train_stream over the text lines
    st = ref_store(F, k, hidden, bits, flat)
    rep = rt.train_stream(iter(text), st, schema)
    ts_final = st.flat.copy()
    ts_version = st.version
    # hogwild_train with one worker (byte-identical to sequential, T:1-11)
    st = ref_store(F, k, hidden, bits, flat)
    hrep = rt.hogwild_train(iter(text), st, schema, rt.TrainOptions(n_threads=1))
    hw_final = st.flat.copy()
    # evaluate_stream on the good lines (+ blank lines) against the trained store
    st = ref_store(F, k, hidden, bits, flat)
    st.flat[:] = ts_final
    ev_lines = [t for t in text if not t.startswith("2 ") and ("|" in t or not t.strip())]
    auc, ll, cnt = rt.evaluate_stream(iter(ev_lines), st, schema)
    series = np.array([(i, np.nan if a is None else a) for i, a in rep.rolling_auc_series])
    np.savez_compressed(os.path.join(HERE, "api.npz"), idx=idx, val=val, labels=labels,
                        F=F, k=k, hidden=np.array(hidden, np.int64), bits=bits, w_seed=133,
                        scale=0.1, flat_sha=sha(flat), names=np.array(names),
                        text=np.array("".join(text)),
                        loop_p=np.array(loop_p), loop_loss=np.array(loop_loss),
                        loop_final=loop_final, loop_version=loop_version,
                        ts_seen=rep.examples_seen, ts_parse_errors=rep.parse_errors,
                        ts_logloss=rep.progressive_logloss, ts_series=series,
                        ts_final=ts_final, ts_version=ts_version,
                        hw_seen=hrep.examples_seen, hw_parse_errors=hrep.parse_errors,
                        hw_logloss=hrep.progressive_logloss, hw_final=hw_final,
                        hw_series=np.array([(i, np.nan if a is None else a)
                                            for i, a in hrep.rolling_auc_series]),
                        ev_auc=np.nan if auc is None else auc, ev_logloss=ll, ev_n=cnt,
                        **keep)
    print("api", n, "examples; parse errors", rep.parse_errors, "logloss",
          rep.progressive_logloss, "eval", auc, ll, cnt)


def main():
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[name + "_fixture"]()
        return
    hash_fixture()
    fwd_fixture("cfg1", configs.CFG1, 256, 10, 101, 0.1)
    fwd_fixture("cfg2", configs.CFG2, 256, 12, 102, 0.05)
    fwd_fixture("cfg5", configs.CFG5, 64, 11, 105, 0.05, bf16=True)
    train_fixture("salted", configs.CFG3, 400, 8, 103, True)
    train_fixture("unsalted", configs.CFG3, 400, 8, 104, False)
    train_fixture("pt025_dense", configs.CFG3, 200, 8, 106, False, power_t=0.25, sparse=False)
    train_fixture("ffm_lr", configs.CFG1, 600, 10, 107, True)
    ctx_fixture()
    metrics_fixture()
    serial_fixture()
    parse_fixture()
    api_fixture()


if __name__ == "__main__":
    main()
