"""K10 GPU text parse (fw_parse_lines / fw_parse_emit) against the reference's
parse_example outputs (tests/golden/parse.npz) and the oracle restatement:
failing lines, labels, field counts and hashed / raw indices bit-exact; values
within 4 f64 ulp (exact on the decimal fast path) and identical once rounded to
the f32 the device model consumes.  Then parsed lines feed K9 + K1."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200.errors import ParseError
from paper_2407_10115_b200.features import InputSchema, parse_lines, split_lines
from tests.golden_io import load

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _check(out, ok, labels, ex_off, cnt_or_fid, idx, val, F, fid_given):
    st = out.status.cpu().numpy()
    assert np.array_equal(st == 0, ok), np.flatnonzero((st == 0) != ok)[:10]
    assert np.array_equal(out.labels.cpu().numpy()[ok], labels[ok])
    b = out.batch
    assert np.array_equal(b.ex_off.cpu().numpy(), ex_off)
    cnt = b.cnt.cpu().numpy().astype(np.int64)
    if fid_given:
        fid = np.repeat(np.tile(np.arange(F), len(ok)), cnt.ravel())
        assert np.array_equal(fid, cnt_or_fid)
    else:
        assert np.array_equal(cnt, cnt_or_fid)
    assert np.array_equal(b.idx.cpu().numpy().astype(np.int64), idx)
    v64 = out.val64.cpu().numpy()
    with np.errstate(over="ignore"):
        ulp = np.abs(v64 - val) / np.maximum(np.spacing(np.abs(val)), 5e-324)
        v32 = val.astype(np.float32)
    assert ulp.max() <= 4, (ulp.max(), v64[ulp.argmax()], val[ulp.argmax()])
    assert np.array_equal(b.val.cpu().numpy(), v32)
    return int((ulp == 0).sum())


def test_parse_matches_reference_golden():
    g = load("parse")
    sc = InputSchema.from_text(str(g["schema"]))
    out = parse_lines(g["text"].tobytes(), sc, DEV, keep_f64=True, raise_on_error=False)
    exact = _check(out, g["ok"], g["labels"], g["ex_off"], g["fid"], g["idx"], g["val"],
                   sc.n_fields, True)
    assert exact >= 0.99 * len(g["val"])


def _random_lines(n, seed):
    rng = np.random.default_rng(seed)
    names = [f"f{i}" for i in range(24)]
    out = []
    for _ in range(n):
        parts = [str(int(rng.integers(0, 2)))]
        for f in rng.permutation(24)[: int(rng.integers(8, 25))]:
            toks = [f"t{int(r)}" for r in rng.zipf(1.3, int(rng.integers(1, 4)))]
            if f >= 20:
                toks = [t + f":{rng.lognormal():.6g}" for t in toks]
            parts.append(f"|{names[f]} " + " ".join(toks))
        out.append(" ".join(parts))
    return names, out


def test_parse_random_lines_match_oracle():
    names, lines = _random_lines(20000, 5)
    sc = InputSchema(tuple(names), frozenset(names[20:]), 24)
    text = ("\n".join(lines) + "\n").encode()
    out = parse_lines(text, sc, DEV, keep_f64=True)
    ok, labels, off, cnt, idx, val = fo.parse_lines_ragged([ln.encode() for ln in lines],
                                                           names, names[20:], 24)
    assert ok.all()
    _check(out, ok, labels, off, cnt, idx, val, 24, False)


def test_parse_errors_raise_at_first_bad_line():
    sc = InputSchema(("a", "b"), frozenset(), 12)
    with pytest.raises(ParseError, match="line 3"):
        parse_lines(b"1 |a x\n0 |b y\n1 |c z\n7 |a\n", sc, DEV)
    out = parse_lines(b"1 |a x\n\n   \n0 |b y\n", sc, DEV)  # blank lines: skipped, no error
    assert out.status.cpu().tolist() == [0, 11, 11, 0]
    assert out.batch.ex_off.cpu().tolist() == [0, 1, 1, 1, 2]
    out = parse_lines("1 |a x y\n".encode(), sc, DEV, raise_on_error=False)
    assert out.status.cpu().tolist() == [8]  # U+00A0 would split in str.split(): rejected
    many = "1 |a " + " ".join(f"t{j}" for j in range(300))  # > 255 in one field: GPU limit
    out = parse_lines((many + "\n1 |b y").encode(), sc, DEV, raise_on_error=False)
    assert out.status.cpu().tolist() == [10, 0]


def test_parsed_lines_feed_the_forward():
    """text -> K10 -> K9 -> K1 equals the oracle forward on the oracle's parse."""
    from paper_2407_10115_b200 import _lib
    from paper_2407_10115_b200.model import ModelConfig, StatusWord, WeightStore, predict_batch
    names, lines = _random_lines(3000, 9)
    bits = 14
    sc = InputSchema(tuple(names), frozenset(names[20:]), bits)
    out = parse_lines(("\n".join(lines)).encode(), sc, DEV)
    b = out.batch
    n, F, M = b.n, b.n_fields, b.max_per_field
    pi = torch.empty((n, F, M), dtype=torch.int32, device=DEV)
    pv = torch.empty((n, F, M), dtype=torch.float32, device=DEV)
    st = StatusWord(DEV)
    st.clear()
    _lib.check(_lib.lib().dffm_unpack_ragged(b.ex_off.data_ptr(), b.cnt.data_ptr(),
                                             b.idx.data_ptr(), b.val.data_ptr(), n, F, M, 0,
                                             pi.data_ptr(), pv.data_ptr(), 0, st.ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    ost = fo.random_store(F, 8, (64, 32), bits, seed=3)
    cfg = ModelConfig(n_fields=F, k=8, hidden_sizes=(64, 32), hash_bits=bits)
    store = WeightStore.from_flat(cfg, ost.flat(False), DEV, "f32", False)
    prob = predict_batch(pi, pv, store).double().cpu().numpy()
    _, ref = fo.forward_batch(pi.cpu().numpy(), pv.cpu().numpy(), ost)
    assert (np.abs(prob - ref) / ref).max() < 1e-5


@pytest.mark.parametrize("chunk", [1, 7, 4096, 1 << 17])
def test_host_text_parser_chunks_match_parse_lines(chunk):
    """HostTextParser (pinned host text, chunked H2D overlapped with K10) gives,
    chunk by chunk, exactly the rows of one parse_lines call: status, labels,
    counts, ragged offsets, indices and values; failed and blank lines included."""
    from paper_2407_10115_b200.features import HostTextParser
    names, lines = _random_lines(9000 if chunk > 1 else 300, 13)
    lines[5] = "7 |f1 x"            # bad label
    lines[17] = "   "                # blank
    lines[-1] = "1 |nofield t"       # unknown field, last line
    sc = InputSchema(tuple(names), frozenset(names[20:]), 20)
    text = ("\n".join(lines) + "\n").encode()
    ref = parse_lines(text, sc, DEV, raise_on_error=False)
    buf, off = split_lines(text)
    h_text = torch.from_numpy(buf.copy()).pin_memory()
    h_off = torch.from_numpy(off).pin_memory()
    st_h = torch.full((len(lines),), -1, dtype=torch.int32).pin_memory()
    p = HostTextParser(sc, DEV, len(lines), len(buf), chunk_lines=chunk)
    for _ in range(2):  # second call reuses every buffer
        parts = p(h_text, h_off, st_h)
        assert [c0 for c0, _, _ in parts] == list(range(0, len(lines), min(chunk, len(lines))))
        assert torch.equal(st_h, ref.status.cpu())
        r_off = ref.batch.ex_off.cpu()
        for c0, c1, pl in parts:
            assert torch.equal(pl.status.cpu(), ref.status[c0:c1].cpu())
            assert torch.equal(pl.labels.cpu(), ref.labels[c0:c1].cpu())
            assert torch.equal(pl.batch.cnt.cpu(), ref.batch.cnt[c0:c1].cpu())
            assert torch.equal(pl.batch.ex_off.cpu(), r_off[c0:c1 + 1] - r_off[c0])
            z0, z1 = int(r_off[c0]), int(r_off[c1])
            assert torch.equal(pl.batch.idx.cpu(), ref.batch.idx[z0:z1].cpu())
            assert torch.equal(pl.batch.val.cpu(), ref.batch.val[z0:z1].cpu())
    with pytest.raises(Exception, match="exceed"):
        HostTextParser(sc, DEV, 10, 100)(h_text, h_off)
