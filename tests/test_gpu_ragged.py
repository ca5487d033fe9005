"""K9 ragged -> padded unpack (dffm_unpack_ragged) and the ragged host-buffer
path (HostPredictor.predict_ragged): bit-exact against the padded layout and
the padded path; contract violations reported at the first bad example."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200 import _lib, configs, synth
from paper_2407_10115_b200.errors import ContractError
from paper_2407_10115_b200.features import PackedBatch, RaggedBatch
from paper_2407_10115_b200.model import HostPredictor, ModelConfig, StatusWord, WeightStore, \
    predict_batch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _unpack(rb, status_base=0):
    n, F, M = rb.n, rb.n_fields, rb.max_per_field
    t = [torch.as_tensor(a).to(DEV) for a in (rb.ex_off, rb.cnt, rb.idx, rb.val)]
    oi = torch.empty((n, F, M), dtype=torch.int32, device=DEV)
    ov = torch.empty((n, F, M), dtype=torch.float32, device=DEV)
    st = StatusWord(DEV)
    st.clear()
    _lib.check(_lib.lib().dffm_unpack_ragged(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(),
                                             t[3].data_ptr(), n, F, M, int(rb.ex_off[0]),
                                             oi.data_ptr(), ov.data_ptr(), status_base, st.ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    st.fetch_async()
    torch.cuda.synchronize()
    return oi.cpu().numpy(), ov.cpu().numpy(), st


@pytest.mark.parametrize("F,M,n", [(24, 3, 5000), (40, 1, 777), (3, 6, 64), (255, 1, 33)])
def test_unpack_ragged_bit_exact(F, M, n):
    rng = np.random.default_rng(F * 31 + M)
    cnt = rng.integers(0, M + 1, size=(n, F))
    cnt[::9] = 0
    idx = np.full((n, F, M), -1, np.int32)
    val = np.zeros((n, F, M), np.float32)
    live = np.arange(M)[None, None, :] < cnt[:, :, None]
    idx[live] = rng.integers(0, 1 << 24, size=int(live.sum()))
    val[live] = rng.lognormal(size=int(live.sum())).astype(np.float32)
    rb = RaggedBatch.from_padded(idx, val)
    oi, ov, st = _unpack(rb)
    st.raise_if_set()
    assert np.array_equal(oi, idx) and np.array_equal(ov.view(np.uint32), val.view(np.uint32))


def test_unpack_ragged_contract_errors():
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 100, size=(50, 4, 2)).astype(np.int32)
    val = np.ones_like(idx, np.float32)
    rb = RaggedBatch.from_padded(idx, val)
    bad = RaggedBatch(rb.ex_off, rb.cnt.copy(), rb.idx, rb.val, 2)
    bad.cnt[23, 1] = 3  # more than max_per_field
    _, _, st = _unpack(bad, status_base=1000)
    with pytest.raises(ContractError) as ei:
        st.raise_if_set()
    assert ei.value.example == 1023
    bad = RaggedBatch(rb.ex_off.copy(), rb.cnt, rb.idx, rb.val, 2)
    bad.ex_off[31:] += 1  # example 30's count sum disagrees with its offsets
    _, _, st = _unpack(bad)
    with pytest.raises(ContractError) as ei:
        st.raise_if_set()
    assert ei.value.example == 30


@pytest.mark.parametrize("wl_name", ["CFG2", "CFG5"])
def test_host_predictor_ragged_equals_padded(wl_name):
    """The ragged host path (K9 + K1, chunked, overlapped copies) returns the
    bits of the padded device run, several chunks with a ragged tail."""
    wl = getattr(configs, wl_name)
    bits = 12
    ost = fo.random_store(wl.n_fields, wl.k, wl.hidden, bits, seed=7, scale=0.05)
    cfg = ModelConfig(n_fields=wl.n_fields, k=wl.k, hidden_sizes=wl.hidden, hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, "bf16" if wl_name == "CFG5" else "f32",
                               False)
    n = 3 * 4096 + 123
    idx, val = synth.make_examples(wl, n, seed=9, hash_bits=bits)
    ref = predict_batch(idx, val, st).cpu()
    rb = RaggedBatch.from_padded(idx.numpy(), val.numpy())
    rbh = RaggedBatch(*(torch.from_numpy(a).pin_memory() for a in (rb.ex_off, rb.cnt, rb.idx,
                                                                  rb.val)), rb.max_per_field)
    hp = HostPredictor(st, n, idx.shape[2], chunk=4096)
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    hp.predict_ragged(rbh, out)
    assert torch.equal(out, ref)
    out2 = torch.empty(n, dtype=torch.float32).pin_memory()
    hp(idx.pin_memory(), val.pin_memory(), out2)
    assert torch.equal(out2, ref)


@pytest.mark.parametrize("wl_name", ["CFG2", "CFG5"])
def test_host_predictor_packed_equals_padded(wl_name):
    """The packed wire format (3-byte indices, 1.0 values elided; K9b) returns
    the bits of the padded device run, several chunks with a ragged tail."""
    wl = getattr(configs, wl_name)
    bits = 20
    ost = fo.random_store(wl.n_fields, wl.k, wl.hidden, bits, seed=8, scale=0.05)
    cfg = ModelConfig(n_fields=wl.n_fields, k=wl.k, hidden_sizes=wl.hidden, hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, "bf16" if wl_name == "CFG5" else "f32",
                               False)
    n = 3 * 4096 + 77
    idx, val = synth.make_examples(wl, n, seed=10, hash_bits=bits)
    ref = predict_batch(idx, val, st).cpu()
    pk = PackedBatch.from_ragged(RaggedBatch.from_padded(idx.numpy(), val.numpy()))
    assert pk.idx_width == 3
    pkh = PackedBatch(*(torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                        for a in (pk.ex_off, pk.cnt, pk.idx_bytes)), 3,
                      *(torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                        for a in (pk.vbits, pk.vals, pk.voff)), pk.max_per_field)
    hp = HostPredictor(st, n, idx.shape[2], chunk=4096)
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    hp.predict_packed(pkh, out)
    assert torch.equal(out, ref)


def test_host_predictor_packed_reports_global_example_index():
    """A non-finite row hit only by an example in a later chunk is reported at
    that example's batch-global index (status_base per chunk), as M:392-396."""
    from paper_2407_10115_b200.errors import NumericError
    wl = configs.CFG2
    bits = 12
    ost = fo.random_store(wl.n_fields, wl.k, wl.hidden, bits, seed=12)
    n = 10_000
    idx, val = synth.make_examples(wl, n, seed=13, hash_bits=bits)
    bad_e = 7_777
    j = int(idx[bad_e, 3, 0])
    ix = idx.numpy().copy()
    ix[:, :, :][ix == j] = -1  # only example bad_e keeps bucket j
    ix[bad_e, 3, 0] = j
    vv = np.where(ix >= 0, val.numpy(), 0).astype(np.float32)
    ost.ffm[j, 5, 0] = np.inf
    cfg = ModelConfig(n_fields=wl.n_fields, k=wl.k, hidden_sizes=wl.hidden, hash_bits=bits)
    st = WeightStore.from_flat(cfg, ost.flat(False), DEV, "f32", False)
    pk = PackedBatch.from_ragged(RaggedBatch.from_padded(ix, vv))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    pkh = PackedBatch(pin(pk.ex_off), pin(pk.cnt), pin(pk.idx_bytes), pk.idx_width,
                      pin(pk.vbits), pin(pk.vals), pin(pk.voff), pk.max_per_field)
    hp = HostPredictor(st, n, ix.shape[2], chunk=2048)
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    with pytest.raises(NumericError) as ei:
        hp.predict_packed(pkh, out)
    assert ei.value.example == bad_e and ei.value.block == "ffm"
