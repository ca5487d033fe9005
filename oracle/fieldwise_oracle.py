"""CPU oracle for the DeepFFM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``fieldwise``
(``/root/reference/pkg/src/fieldwise``), used as the *checker* by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  Nothing in the product package
(``paper_2407_10115_b200``) imports it; the product fails loudly without its
CUDA library instead of falling back here.

Pinning.  The rows that restate code present in the reference (forward,
backward_update, Adagrad, duplicate merge, hashing) are pinned against golden
vectors produced by running the reference itself (``tests/golden/
make_golden.py`` -> ``tests/golden/*.npz``; checked by
``tests/test_oracle_golden.py``).  Quantisation and context caching exist only
in SPEC.md; for them the oracle follows SPEC with the
precision choices pinned in SURVEY.md section 8(a) row Q, and the SPEC
known-answer examples are the only external pins ("parity unpinned" beyond
those KATs).

Reference citations use ``M:`` = model.py, ``Fe:`` = features.py,
``H:`` = hashing.py, ``S:`` = SPEC.md line numbers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MERGE_EPS = 1e-6  # M:37
PROB_CLAMP = 1e-7  # M:38
FNV32_OFFSET = 0x811C9DC5  # H:15
FNV32_PRIME = 0x01000193  # H:16
FIELD_TOKEN_SEP = b"\x1f"  # H:22


class OracleNumericError(Exception):
    def __init__(self, msg, block):
        super().__init__(msg)
        self.block = block


# --------------------------------------------------------------------------
# pair order (M:113-127)
# --------------------------------------------------------------------------


def pair_indices(n_fields: int):
    """Strict upper triangle, row-major: (0,1),(0,2),...  (M:113-117)."""
    iu, ju = np.triu_indices(n_fields, k=1)
    return iu.astype(np.int64), ju.astype(np.int64)


# --------------------------------------------------------------------------
# weight store (M:142-230): separate f32 blocks + the frozen flat layout
# --------------------------------------------------------------------------


@dataclass
class OracleStore:
    n_fields: int
    k: int
    hidden_sizes: tuple
    hash_bits: int
    lr: np.ndarray  # f32 [2^b + 1], bias at the end (M:148-149)
    ffm: np.ndarray  # f32 [2^b, F, k] (M:150-151)
    layers: list  # [(W f32 [in,out], b f32 [out])] (M:152)
    lr_acc: np.ndarray = None
    ffm_acc: np.ndarray = None
    layer_accs: list = field(default_factory=list)

    @property
    def n_features(self):
        return 1 << self.hash_bits

    @property
    def n_pairs(self):
        return self.n_fields * (self.n_fields - 1) // 2

    @property
    def nn_dims(self):
        if not self.hidden_sizes:
            return []
        dims = [1 + self.n_pairs, *self.hidden_sizes, 1]
        return list(zip(dims[:-1], dims[1:]))

    @classmethod
    def zeros(cls, n_fields, k, hidden_sizes, hash_bits):
        nb = 1 << hash_bits
        hidden_sizes = tuple(int(h) for h in hidden_sizes)
        st = cls(n_fields, k, hidden_sizes, hash_bits,
                 np.zeros(nb + 1, np.float32), np.zeros((nb, n_fields, k), np.float32), [])
        for i, o in st.nn_dims:
            st.layers.append((np.zeros((i, o), np.float32), np.zeros(o, np.float32)))
        st.lr_acc = np.ones_like(st.lr)  # acc0 = 1.0 (M:271)
        st.ffm_acc = np.ones_like(st.ffm)
        st.layer_accs = [(np.ones_like(w), np.ones_like(b)) for w, b in st.layers]
        return st

    def copy(self):
        return OracleStore(
            self.n_fields, self.k, self.hidden_sizes, self.hash_bits,
            self.lr.copy(), self.ffm.copy(), [(w.copy(), b.copy()) for w, b in self.layers],
            self.lr_acc.copy(), self.ffm_acc.copy(),
            [(w.copy(), b.copy()) for w, b in self.layer_accs])

    def flat(self, include_optimizer=True) -> np.ndarray:
        """Frozen flat order lr -> ffm -> (W,b)* -> accumulators (M:145-153)."""
        parts = [self.lr, self.ffm.ravel()]
        for w, b in self.layers:
            parts += [w.ravel(), b]
        if include_optimizer:
            parts += [self.lr_acc, self.ffm_acc.ravel()]
            for w, b in self.layer_accs:
                parts += [w.ravel(), b]
        return np.concatenate(parts).astype(np.float32)

    @classmethod
    def from_flat(cls, n_fields, k, hidden_sizes, hash_bits, flat):
        st = cls.zeros(n_fields, k, hidden_sizes, hash_bits)
        flat = np.asarray(flat, np.float32)
        off = 0

        def take(n):
            nonlocal off
            out = flat[off:off + n].copy()
            off += n
            return out

        st.lr = take(st.lr.size)
        st.ffm = take(st.ffm.size).reshape(st.ffm.shape)
        st.layers = [(take(i * o).reshape(i, o), take(o)) for i, o in st.nn_dims]
        if off < flat.size:
            st.lr_acc = take(st.lr.size)
            st.ffm_acc = take(st.ffm.size).reshape(st.ffm.shape)
            st.layer_accs = [(take(i * o).reshape(i, o), take(o)) for i, o in st.nn_dims]
        return st


def random_store(n_fields, k, hidden_sizes, hash_bits, seed, scale=0.05, acc=1.0):
    """N(0, scale) f32 weights drawn in flat-layout order (SURVEY 8(d) cfg2/3 recipe)."""
    st = OracleStore.zeros(n_fields, k, hidden_sizes, hash_bits)
    rng = np.random.default_rng(seed)
    st.lr[:] = (rng.standard_normal(st.lr.size) * scale).astype(np.float32)
    st.ffm[:] = (rng.standard_normal(st.ffm.size) * scale).astype(np.float32).reshape(st.ffm.shape)
    for w, b in st.layers:
        w[:] = (rng.standard_normal(w.size) * scale).astype(np.float32).reshape(w.shape)
        b[:] = (rng.standard_normal(b.size) * scale).astype(np.float32)
    for a in [st.lr_acc, st.ffm_acc] + [x for wb in st.layer_accs for x in wb]:
        a[...] = acc
    return st


# --------------------------------------------------------------------------
# canonical example form (Fe:121-172) <-> padded GPU arrays
# --------------------------------------------------------------------------


def row_to_fields(idx_row, val_row):
    """Padded [F][M] row (sentinel -1) -> [(field_id, int64 idx, f64 val)].

    Field order = ascending field id (the GPU layout); within a field the
    indices are strictly increasing with duplicate values summed (Fe:166-172,
    Fe:219)."""
    out = []
    for f in range(idx_row.shape[0]):
        sel = idx_row[f] >= 0
        if not sel.any():
            continue
        ix = idx_row[f][sel].astype(np.int64)
        vx = val_row[f][sel].astype(np.float64)
        u, inv = np.unique(ix, return_inverse=True)
        if len(u) != len(ix):
            vv = np.zeros(len(u))
            np.add.at(vv, inv, vx)
            ix, vx = u, vv
        else:
            order = np.argsort(ix, kind="stable")
            ix, vx = ix[order], vx[order]
        out.append((f, ix, vx))
    return out


# --------------------------------------------------------------------------
# forward (M:293-397)
# --------------------------------------------------------------------------


def sigmoid(logit: float) -> float:
    """Stable sigmoid with +-60 clamp (M:293-297)."""
    if logit >= 0:
        return 1.0 / (1.0 + math.exp(-min(logit, 60.0)))
    e = math.exp(max(logit, -60.0))
    return e / (1.0 + e)


def predict_proba(logit: float) -> float:
    """Clamped probability (M:300-305)."""
    if not math.isfinite(logit):
        raise OracleNumericError("non-finite logit", "logit")
    p = sigmoid(logit)
    return min(max(p, PROB_CLAMP), 1.0 - PROB_CLAMP)


def forward(fields, st: OracleStore, mac=None):
    """One example through lr -> ffm -> merge -> mlp (M:321-397).

    ``fields``: list of (field_id, int64 indices, f64 values).  Returns a dict
    holding the intermediates ``backward_update`` needs (M:275-290)."""
    F, k = st.n_fields, st.k
    lr_out = float(st.lr[st.n_features])  # M:327
    s = np.zeros((F, F, k))
    present = np.zeros(F, dtype=bool)
    for fid, ix, vx in fields:
        if fid >= F:
            raise ValueError("field id outside model")  # M:331-334 (ContractError)
        m = len(ix)
        if m == 0:
            continue
        lr_out += float(np.dot(st.lr[ix], vx))  # M:338
        s[fid] += np.tensordot(vx, st.ffm[ix], axes=(0, 0))  # M:339
        present[fid] = True
        if mac is not None:
            mac[0] += m + m * F * k  # M:341-342
    iu, ju = pair_indices(F)
    pair_out = np.zeros(st.n_pairs)
    active = present[iu] & present[ju]
    if active.any():
        pair_out[active] = np.einsum("ak,ak->a", s[iu[active], ju[active]], s[ju[active], iu[active]])
        if mac is not None:
            mac[0] += int(active.sum()) * k  # M:352-353
    v = np.empty(1 + st.n_pairs)
    v[0] = lr_out
    v[1:] = pair_out
    mu = float(v.mean())
    sd = float(v.std())
    merged = (v - mu) / (sd + MERGE_EPS)  # M:355-360
    pre, acts = [], []
    nn_out = 0.0
    if st.layers:
        a = merged
        for w, b in st.layers[:-1]:
            z = a @ w + b  # M:367-371
            pre.append(z)
            a = np.maximum(z, 0.0)
            acts.append(a)
        w_out, b_out = st.layers[-1]
        nn_out = float(a @ w_out[:, 0] + b_out[0])  # M:372-373
        if mac is not None:
            mac[0] += sum(i * o for i, o in st.nn_dims)
    logit = nn_out + lr_out + float(pair_out.sum())  # M:377
    state = dict(lr_out=lr_out, pairs=pair_out, merged=merged, pre=pre, acts=acts,
                 logit=logit, s=s, v=v, mu=mu, sd=sd, nn_out=nn_out)
    if not math.isfinite(logit):
        raise OracleNumericError("non-finite", diagnose_nonfinite(state))
    return state


def diagnose_nonfinite(state) -> str:
    """First non-finite block in lr -> ffm -> merge -> nn -> logit (M:308-318)."""
    if not math.isfinite(state["lr_out"]):
        return "lr"
    if not np.isfinite(state["pairs"]).all():
        return "ffm"
    if not np.isfinite(state["merged"]).all():
        return "merge"
    for z in state["pre"]:
        if not np.isfinite(z).all():
            return "nn"
    return "logit"


def forward_batch(idx, val, st: OracleStore, chunk=2048):
    """Vectorised fp64 restatement of ``forward`` over padded arrays.

    Same math as M:321-377; summation order differs from the per-example
    loop only at the 1e-16 level.  Returns (logit f64 [n], prob f64 [n])."""
    idx = np.asarray(idx)
    val = np.asarray(val)
    n, F, M = idx.shape
    k = st.k
    iu, ju = pair_indices(F)
    logits = np.empty(n)
    ffm64 = None
    for c0 in range(0, n, chunk):
        ix = idx[c0:c0 + chunk].astype(np.int64)
        vx = val[c0:c0 + chunk].astype(np.float64)
        ok = ix >= 0
        safe = np.where(ok, ix, 0)
        x = np.where(ok, vx, 0.0)
        lr_out = float(st.lr[st.n_features]) + (st.lr[safe].astype(np.float64) * x).sum(axis=(1, 2))
        rows = st.ffm[safe].astype(np.float64)  # [c,F,M,F,k]
        s = np.einsum("cfm,cfmgk->cfgk", x, rows)
        present = ok.any(axis=2)
        act = present[:, iu] & present[:, ju]
        pairs = np.einsum("cpk,cpk->cp", s[:, iu, ju], s[:, ju, iu]) * act
        v = np.concatenate([lr_out[:, None], pairs], axis=1)
        mu = v.mean(axis=1, keepdims=True)
        sd = v.std(axis=1, keepdims=True)
        merged = (v - mu) / (sd + MERGE_EPS)
        nn_out = 0.0
        if st.layers:
            a = merged
            for w, b in st.layers[:-1]:
                a = np.maximum(a @ w.astype(np.float64) + b, 0.0)
            w_out, b_out = st.layers[-1]
            nn_out = a @ w_out[:, 0].astype(np.float64) + float(b_out[0])
        logits[c0:c0 + chunk] = nn_out + lr_out + pairs.sum(axis=1)
    p = 1.0 / (1.0 + np.exp(-np.clip(logits, -60.0, 60.0)))
    return logits, np.clip(p, PROB_CLAMP, 1.0 - PROB_CLAMP)


# --------------------------------------------------------------------------
# backward + Adagrad (M:400-572)
# --------------------------------------------------------------------------


def _inv_pow(acc, power_t):
    if power_t == 0.5:  # M:400-404
        return 1.0 / np.sqrt(acc)
    return np.power(acc, -power_t)


def _inv_pow_scalar(acc, power_t):
    if power_t == 0.5:  # M:407-410
        return 1.0 / math.sqrt(acc)
    return acc ** -power_t


def _merge_backward(state, d_merged):
    """MergeNorm Jacobian (M:413-421)."""
    v = state["v"]
    d = len(v)
    denom = state["sd"] + MERGE_EPS
    dv = (d_merged - d_merged.mean()) / denom
    if state["sd"] > 0.0:
        c = v - state["mu"]
        dv = dv - c * (float(np.dot(d_merged, c)) / (d * state["sd"] * denom * denom))
    return dv


def _merge_unique(indices, grads):
    """Sort-and-segment duplicate merge in occurrence order (M:424-437)."""
    uidx, inverse = np.unique(indices, return_inverse=True)
    if len(uidx) == len(indices):
        return uidx, grads[np.argsort(indices)]
    merged = np.zeros((len(uidx),) + grads.shape[1:])
    np.add.at(merged, inverse, grads)
    return uidx, merged


def _update_matrix(w, w_acc, a_in, d, lr, pt, sparse):
    """M:536-554."""
    if sparse:
        rows = np.flatnonzero(a_in)
        cols = np.flatnonzero(d)
        if len(rows) == 0 or len(cols) == 0:
            return
        if len(rows) < len(a_in) or len(cols) < len(d):
            ix = np.ix_(rows, cols)
            grad = np.outer(a_in[rows], d[cols])
            acc = w_acc[ix].astype(np.float64)
            acc += grad * grad
            w_acc[ix] = acc
            w[ix] = w[ix] - lr * grad * _inv_pow(acc, pt)
            return
    grad = np.outer(a_in, d)
    acc = w_acc.astype(np.float64)
    acc += grad * grad
    w_acc[...] = acc
    w[...] = w - lr * grad * _inv_pow(acc, pt)


def _update_bias(b, b_acc, d, lr, pt, sparse):
    """M:557-572."""
    if sparse:
        cols = np.flatnonzero(d)
        if len(cols) == 0:
            return
        if len(cols) < len(d):
            grad = d[cols]
            acc = b_acc[cols].astype(np.float64)
            acc += grad * grad
            b_acc[cols] = acc
            b[cols] = b[cols] - lr * grad * _inv_pow(acc, pt)
            return
    acc = b_acc.astype(np.float64)
    acc += d * d
    b_acc[...] = acc
    b[...] = b - lr * d * _inv_pow(acc, pt)


def backward_update(state, fields, label, st: OracleStore, lr_ffm, lr_lr, lr_nn, power_t,
                    sparse=True):
    """One Adagrad step in place; returns the example's log-loss (M:440-533)."""
    if label not in (0, 1):
        raise ValueError("label must be 0 or 1")  # M:453-454
    p_raw = sigmoid(state["logit"])
    g = p_raw - label  # M:456-457
    if not math.isfinite(g):
        raise OracleNumericError("non-finite loss gradient", "loss")
    p = min(max(p_raw, PROB_CLAMP), 1.0 - PROB_CLAMP)
    loss = -math.log(p) if label else -math.log1p(-p)
    pt = power_t
    F, k = st.n_fields, st.k
    if st.layers:
        d = np.array([g])
        inputs = [state["merged"]] + state["acts"]
        for i in range(len(st.layers) - 1, -1, -1):
            a_in = inputs[i]
            w, b = st.layers[i]
            w_acc, b_acc = st.layer_accs[i]
            da_in = w @ d  # pre-update weights (M:473-475)
            _update_matrix(w, w_acc, a_in, d, lr_nn, pt, sparse)
            _update_bias(b, b_acc, d, lr_nn, pt, sparse)
            if i > 0:
                d = da_in * (state["pre"][i - 1] > 0.0)  # M:479
            else:
                d_merged = da_in
        dv = _merge_backward(state, d_merged)
        d_lr = g + float(dv[0])  # M:483
        d_pairs = g + dv[1:]  # M:484
    else:
        d_lr = g
        d_pairs = np.full(st.n_pairs, g)
    if st.n_pairs:
        dp = np.zeros((F, F))
        iu, ju = pair_indices(F)
        dp[iu, ju] = d_pairs
        dp[ju, iu] = d_pairs
        idx_parts, grad_parts = [], []
        for fid, ix, vx in fields:
            if len(ix) == 0:
                continue
            t = dp[fid][:, None] * state["s"][:, fid, :]  # M:501
            if not t.any():
                continue  # M:502
            idx_parts.append(ix)
            grad_parts.append(vx[:, None, None] * t[None, :, :])
        if idx_parts:
            uidx, ug = _merge_unique(np.concatenate(idx_parts), np.concatenate(grad_parts))
            acc = st.ffm_acc[uidx].astype(np.float64)
            acc += ug * ug
            st.ffm_acc[uidx] = acc
            st.ffm[uidx] = st.ffm[uidx] - lr_ffm * ug * _inv_pow(acc, pt)  # M:509-513
    idx_parts = [ix for _, ix, _ in fields if len(ix)]
    if idx_parts:
        vals = np.concatenate([vx for _, ix, vx in fields if len(ix)])
        uidx, ug = _merge_unique(np.concatenate(idx_parts), d_lr * vals)
        acc = st.lr_acc[uidx].astype(np.float64)
        acc += ug * ug
        st.lr_acc[uidx] = acc
        st.lr[uidx] = st.lr[uidx] - lr_lr * ug * _inv_pow(acc, pt)  # M:516-524
    bias = st.n_features
    acc_b = float(st.lr_acc[bias]) + d_lr * d_lr
    st.lr_acc[bias] = acc_b
    st.lr[bias] = float(st.lr[bias]) - lr_lr * d_lr * _inv_pow_scalar(acc_b, pt)  # M:525-530
    return loss


def train_sequential(idx, val, labels, st: OracleStore, lr_ffm, lr_lr, lr_nn, power_t,
                     sparse=True):
    """Predict-then-learn over padded arrays in order (T:172-185).

    Returns (clamped probabilities f64 [n], losses f64 [n])."""
    n = idx.shape[0]
    probs = np.empty(n)
    losses = np.empty(n)
    for e in range(n):
        fields = row_to_fields(idx[e], val[e])
        state = forward(fields, st)
        probs[e] = predict_proba(state["logit"])
        losses[e] = backward_update(state, fields, int(labels[e]), st, lr_ffm, lr_lr, lr_nn,
                                    power_t, sparse)
    return probs, losses


# --------------------------------------------------------------------------
# 16-bit quantisation (precision pinned per
# SURVEY 8(a) row Q)
# --------------------------------------------------------------------------

B_MAX = 65536


def quant_header(wmin: float, wmax: float, alpha: int = 4, beta: int = 4):
    """(w_min_r f32, bucket f32) from the f32 min/max of a table.

    max rounded UP at alpha decimals, min DOWN at beta decimals, in f64
    (S:316); bucket = (max_r - min_r)/65536; both header fields are
    then rounded to f32.  bucket is exactly 0 iff max_r == min_r
    (S:320)."""
    sa = 10.0 ** alpha
    sb = 10.0 ** beta
    max_r = math.ceil(float(np.float64(wmax)) * sa) / sa
    min_r = math.floor(float(np.float64(wmin)) * sb) / sb
    bucket = 0.0 if max_r == min_r else (max_r - min_r) / B_MAX
    return np.float32(min_r), np.float32(bucket)


def quantize(w, alpha=4, beta=4):
    """-> (w_min f32, bucket f32, u16 indices).

    idx = clamp(round_half_even((f64(w) - f64(hmin)) / f64(hbucket)), 0, 65535)
    computed from the f32 header values."""
    w = np.asarray(w, np.float32)
    if w.size == 0:
        raise ValueError("empty input")  # S:317 contract error
    if not np.isfinite(w).all():
        raise OracleNumericError("non-finite weight", "quantize")
    hmin, hb = quant_header(float(w.min()), float(w.max()), alpha, beta)
    if hb == 0.0:
        return hmin, hb, np.zeros(w.shape, np.uint16)
    raw = np.rint((w.astype(np.float64) - np.float64(hmin)) / np.float64(hb))
    return hmin, hb, np.clip(raw, 0, B_MAX - 1).astype(np.uint16)


def dequantize(hmin, hb, q):
    """w' = hmin + idx*bucket, an f32 multiply then an f32 add, each rounded
    to nearest (no fused multiply-add)."""
    prod = (np.asarray(q).astype(np.float32) * np.float32(hb)).astype(np.float32)
    return (np.float32(hmin) + prod).astype(np.float32)


# --------------------------------------------------------------------------
# context cache; truth = forward on the merged example
# --------------------------------------------------------------------------


def build_context_cache(ctx_fields, st: OracleStore, mac=None):
    """lr partial, context latent sums S[x][g] and ctx x ctx pairs."""
    F, k = st.n_fields, st.k
    lr_part = 0.0
    s = np.zeros((F, F, k))
    present = np.zeros(F, bool)
    for fid, ix, vx in ctx_fields:
        if len(ix) == 0:
            continue
        lr_part += float(np.dot(st.lr[ix], vx))
        s[fid] += np.tensordot(vx, st.ffm[ix], axes=(0, 0))
        present[fid] = True
        if mac is not None:
            mac[0] += len(ix) + len(ix) * F * k
    iu, ju = pair_indices(F)
    pairs = np.zeros(st.n_pairs)
    act = present[iu] & present[ju]
    if act.any():
        pairs[act] = np.einsum("ak,ak->a", s[iu[act], ju[act]], s[ju[act], iu[act]])
        if mac is not None:
            mac[0] += int(act.sum()) * k
    return dict(lr_part=lr_part, s=s, present=present, pairs=pairs)


def predict_with_cache(cache, cand_fields, st: OracleStore, mac=None):
    """Finish one candidate from a context cache -> (logit, prob)."""
    F, k = st.n_fields, st.k
    lr_out = float(st.lr[st.n_features]) + cache["lr_part"]
    s = cache["s"].copy()
    present = cache["present"].copy()
    cpresent = np.zeros(F, bool)
    for fid, ix, vx in cand_fields:
        if len(ix) == 0:
            continue
        lr_out += float(np.dot(st.lr[ix], vx))
        s[fid] += np.tensordot(vx, st.ffm[ix], axes=(0, 0))
        cpresent[fid] = True
        if mac is not None:
            mac[0] += len(ix) + len(ix) * F * k
    present |= cpresent
    iu, ju = pair_indices(F)
    pairs = cache["pairs"].copy()
    act = present[iu] & present[ju] & (cpresent[iu] | cpresent[ju])
    if act.any():
        pairs[act] = np.einsum("ak,ak->a", s[iu[act], ju[act]], s[ju[act], iu[act]])
        if mac is not None:
            mac[0] += int(act.sum()) * k
    v = np.concatenate([[lr_out], pairs])
    mu, sd = float(v.mean()), float(v.std())
    merged = (v - mu) / (sd + MERGE_EPS)
    nn_out = 0.0
    if st.layers:
        a = merged
        for w, b in st.layers[:-1]:
            a = np.maximum(a @ w + b, 0.0)
        w_out, b_out = st.layers[-1]
        nn_out = float(a @ w_out[:, 0] + b_out[0])
        if mac is not None:
            mac[0] += sum(i * o for i, o in st.nn_dims)
    logit = nn_out + lr_out + float(pairs.sum())
    return logit, predict_proba(logit)


# --------------------------------------------------------------------------
# hashing (H:28-50)
# --------------------------------------------------------------------------


def fnv1a32(data: bytes) -> int:
    h = FNV32_OFFSET
    for b in data:
        h = ((h ^ b) * FNV32_PRIME) & 0xFFFFFFFF
    return h


def hash_feature(field_name: str, token: str, hash_bits: int) -> int:
    data = field_name.encode("utf-8") + FIELD_TOKEN_SEP + token.encode("utf-8")
    return fnv1a32(data) & ((1 << hash_bits) - 1)


def fnv1a32_batch(blob: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Vectorised FNV-1a over a packed byte buffer (item i = blob[off[i]:off[i+1]])."""
    blob = np.asarray(blob, np.uint8)
    offsets = np.asarray(offsets, np.int64)
    n = len(offsets) - 1
    lens = np.diff(offsets)
    h = np.full(n, FNV32_OFFSET, np.uint64)
    maxlen = int(lens.max()) if n else 0
    for pos in range(maxlen):
        live = lens > pos
        b = blob[offsets[:-1][live] + pos].astype(np.uint64)
        h[live] = ((h[live] ^ b) * np.uint64(FNV32_PRIME)) & np.uint64(0xFFFFFFFF)
    return h.astype(np.uint32)


# --------------------------------------------------------------------------
# weight transfer: varints and FWP1 byte patches (SPEC S:329-353, S:358-362,
# S:381-382).  No reference code exists; pinned by the SPEC examples
# and the declared choices below:
#   * FWP1 header = magic, version u32 (= 1), source digest u64, target
#     digest u64, target length u64, all little-endian
#   * digest = FNV-1a 64 over the full byte content
#   * a byte at offset i < len(new) differs if i >= len(old) or old[i] != new[i];
#     differing runs separated by fewer than GAP_MERGE = 4 identical bytes are
#     merged into one op; `skip` is relative to the END of the
#     previous op (0 for the first), `length` counts payload bytes
#   * apply: output = old[:target_length] zero-extended, ops written in order
# --------------------------------------------------------------------------

FNV64_OFFSET = 0xCBF29CE484222325
FNV64_PRIME = 0x100000001B3
PATCH_MAGIC = b"FWP1"
PATCH_VERSION = 1
GAP_MERGE = 4


class OracleFormatError(Exception):
    pass


class OracleStaleBaseError(Exception):
    pass


class OracleCorruptionError(Exception):
    pass


def fnv1a64(data) -> int:
    h = FNV64_OFFSET
    for b in bytes(data):
        h = ((h ^ b) * FNV64_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def encode_varint(n: int) -> bytes:
    """LEB128: 7-bit groups, little-endian, high bit = continuation."""
    if n < 0 or n >= 1 << 64:
        raise ValueError("varint out of range")
    out = bytearray()
    while True:
        b = n & 0x7F
        n >>= 7
        if n:
            out.append(b | 0x80)
        else:
            out.append(b)
            return bytes(out)


def decode_varint(buf, pos: int = 0):
    """-> (value, bytes consumed); more than 10 bytes or truncation is a format error."""
    n = 0
    shift = 0
    for i in range(10):
        if pos + i >= len(buf):
            raise OracleFormatError("truncated varint")
        b = buf[pos + i]
        n |= (b & 0x7F) << shift
        if not b & 0x80:
            if n >= 1 << 64:
                raise OracleFormatError("varint overflow")
            return n, i + 1
        shift += 7
    raise OracleFormatError("varint longer than 10 bytes")


def diff_ops(old, new):
    """Ordered (start, end_exclusive) ranges of the ops create_patch emits."""
    old = np.frombuffer(bytes(old), np.uint8)
    new = np.frombuffer(bytes(new), np.uint8)
    m = min(len(old), len(new))
    d = np.ones(len(new), bool)
    d[:m] = old[:m] != new[:m]
    pos = np.flatnonzero(d)
    if len(pos) == 0:
        return []
    gaps = np.diff(pos) - 1
    cut = np.flatnonzero(gaps >= GAP_MERGE)
    starts = np.concatenate([[pos[0]], pos[cut + 1]])
    ends = np.concatenate([pos[cut], [pos[-1]]]) + 1
    return list(zip(starts.tolist(), ends.tolist()))


def create_patch(old, new) -> bytes:
    old, new = bytes(old), bytes(new)
    out = bytearray(PATCH_MAGIC)
    out += int(PATCH_VERSION).to_bytes(4, "little")
    out += fnv1a64(old).to_bytes(8, "little") + fnv1a64(new).to_bytes(8, "little")
    out += len(new).to_bytes(8, "little")
    prev = 0
    for a, b in diff_ops(old, new):
        out += encode_varint(a - prev) + encode_varint(b - a) + new[a:b]
        prev = b
    return bytes(out)


def apply_patch(old, patch) -> bytes:
    old, patch = bytes(old), bytes(patch)
    if len(patch) < 32 or patch[:4] != PATCH_MAGIC:
        raise OracleFormatError("not a patch")
    if int.from_bytes(patch[4:8], "little") != PATCH_VERSION:
        raise OracleFormatError("unsupported patch version")
    src = int.from_bytes(patch[8:16], "little")
    dst = int.from_bytes(patch[16:24], "little")
    tlen = int.from_bytes(patch[24:32], "little")
    if fnv1a64(old) != src:
        raise OracleStaleBaseError("source digest mismatch")
    out = bytearray(old[:tlen]) + bytearray(max(0, tlen - len(old)))
    pos, cur = 32, 0
    while pos < len(patch):
        skip, c1 = decode_varint(patch, pos)
        pos += c1
        ln, c2 = decode_varint(patch, pos)
        pos += c2
        start = cur + skip
        if start + ln > tlen:
            raise OracleFormatError("op overruns target length")
        if pos + ln > len(patch):
            raise OracleFormatError("truncated payload")
        out[start:start + ln] = patch[pos:pos + ln]
        pos += ln
        cur = start + ln
    if fnv1a64(out) != dst:
        raise OracleCorruptionError("target digest mismatch")
    return bytes(out)


# text parsing (Fe:1-235) -- checker for K10 (fw_parse_lines)
# --------------------------------------------------------------------------


class OracleParseError(Exception):
    pass


# str.split() / str.strip() whitespace restricted to ASCII (Fe:190, Fe:222: the
# K10 contract rejects lines holding non-ASCII bytes that could decode to
# Unicode whitespace; every ASCII byte str.isspace() accepts is here)
ASCII_WS = b" \t\n\r\x0b\x0c\x1c\x1d\x1e\x1f"


def _split_ws(b: bytes):
    out, cur = [], bytearray()
    for c in b:
        if c in ASCII_WS:
            if cur:
                out.append(bytes(cur))
                cur = bytearray()
        else:
            cur.append(c)
    if cur:
        out.append(bytes(cur))
    return out


def parse_line(line: bytes, field_names, numeric, hash_bits: int):
    """Restatement of parse_example (Fe:221-235) + _parse_blocks (Fe:175-219)
    over the line's UTF-8 bytes.  Returns (label, {field_id: {index: value}})
    with fields in first-appearance order; raises OracleParseError where the
    reference raises ParseError."""
    ids = {n.encode("utf-8"): i for i, n in enumerate(field_names)}
    numeric = {n.encode("utf-8") for n in numeric}
    segs = line.split(b"|")
    head = segs[0].strip(ASCII_WS)
    if head == b"1":
        label = 1
    elif head in (b"0", b"-1"):
        label = 0
    else:
        raise OracleParseError("malformed label")  # Fe:229
    if len(segs) < 2:
        raise OracleParseError("no field blocks")  # Fe:231
    max_index = 1 << hash_bits
    per = {}
    for seg in segs[1:]:
        atoms = _split_ws(seg)
        if not atoms:
            raise OracleParseError("empty field block")  # Fe:191
        name = atoms[0]
        if name not in ids:
            raise OracleParseError("unknown field")  # InputSchema.field_id
        fid = ids[name]
        feats = per.setdefault(fid, {})
        for atom in atoms[1:]:
            token, sep, raw = atom.partition(b":")
            if sep:
                try:
                    value = float(raw.decode("utf-8"))  # Fe:201
                except (ValueError, UnicodeDecodeError):
                    raise OracleParseError("bad value") from None
                if not math.isfinite(value):
                    raise OracleParseError("non-finite value")
            else:
                value = 1.0
            if token.startswith(b"@") and len(token) > 1 and token[1:].isdigit():
                index = int(token[1:])  # Fe:209-214
                if index >= max_index:
                    raise OracleParseError("raw index out of range")
            else:
                index = fnv1a32(name + FIELD_TOKEN_SEP + token) & (max_index - 1)  # H:43-50
                if name in numeric:
                    value = math.log1p(value) if value > 0 else value  # Fe:33-39
            feats[index] = feats.get(index, 0.0) + value  # Fe:219
    return label, per


def parse_lines_ragged(lines, field_names, numeric, hash_bits: int):
    """Lines -> (ok [n] bool, labels [n], ex_off [n+1], cnt [n,F], idx [nnz], val64 [nnz]):
    the canonical features of every parsable line in field-id order, indices
    ascending within a field (the layout K10 writes); failed lines hold none."""
    F = len(field_names)
    n = len(lines)
    ok = np.zeros(n, bool)
    labels = np.zeros(n, np.uint8)
    cnt = np.zeros((n, F), np.int64)
    idx, val, off = [], [], [0]
    for i, ln in enumerate(lines):
        try:
            lab, per = parse_line(ln, field_names, numeric, hash_bits)
        except OracleParseError:
            off.append(off[-1])
            continue
        ok[i] = True
        labels[i] = lab
        for fid in sorted(per):
            items = sorted(per[fid].items())
            cnt[i, fid] = len(items)
            idx += [k for k, _ in items]
            val += [v for _, v in items]
        off.append(len(idx))
    return (ok, labels, np.array(off, np.int64), cnt, np.array(idx, np.int64),
            np.array(val, np.float64))
