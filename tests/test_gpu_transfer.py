"""K7 FWP1 patches: GPU diff/encode/apply vs the oracle
restatement, SPEC examples, fuzzed round trips, error classes, and the
quantised update pipeline."""

import numpy as np
import pytest
import torch

from oracle import fieldwise_oracle as fo
from paper_2407_10115_b200 import transfer
from paper_2407_10115_b200.errors import CorruptionError, FormatError, StaleBaseError
from paper_2407_10115_b200.model import ModelConfig, WeightStore

pytestmark = pytest.mark.gpu


def test_spec_examples():
    p = transfer.create_patch(bytes([1, 2, 3, 4]), bytes([1, 2, 9, 4]))
    assert p == fo.create_patch(bytes([1, 2, 3, 4]), bytes([1, 2, 9, 4]))
    assert p[32:] == bytes([2, 1, 9])  # one op {skip 2, length 1, payload [9]}
    assert transfer.apply_patch(bytes([1, 2, 3, 4]), p) == bytes([1, 2, 9, 4])
    same = transfer.create_patch(b"abcdef", b"abcdef")
    assert len(same) == 32 and transfer.apply_patch(b"abcdef", same) == b"abcdef"


def mutate(rng, old):
    new = bytearray(old)
    for _ in range(int(rng.integers(0, 12))):
        if not new:
            break
        a = int(rng.integers(0, len(new)))
        ln = int(rng.integers(1, 9))
        new[a:a + ln] = rng.integers(0, 256, min(ln, len(new) - a), dtype=np.uint8).tobytes()
    r = rng.random()
    if r < 0.2:
        new += rng.integers(0, 256, int(rng.integers(1, 300)), dtype=np.uint8).tobytes()
    elif r < 0.4 and new:
        del new[int(rng.integers(0, len(new))):]
    return bytes(new)


def test_fuzz_matches_oracle_and_round_trips():
    rng = np.random.default_rng(7)
    for case in range(1500):
        n = int(rng.choice([0, 1, 5, 17, 64, 1000, 4096, 65536]))
        old = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        new = mutate(rng, old) if rng.random() < 0.9 else \
            rng.integers(0, 256, int(rng.integers(0, 70000)), dtype=np.uint8).tobytes()
        p = transfer.create_patch(old, new)
        if n <= 4096 and len(new) <= 4096:  # the oracle's Python digest is slow
            assert p == fo.create_patch(old, new), case
        else:  # op stream from the oracle's diff, header digests from the library
            ops = fo.diff_ops(old, new)
            ref = b"".join(fo.encode_varint(a - (ops[i - 1][1] if i else 0)) + fo.encode_varint(b - a)
                           + new[a:b] for i, (a, b) in enumerate(ops))
            assert p[32:] == ref, case
        assert transfer.apply_patch(old, p) == new, case


def test_sparse_edits_patch_is_small():
    rng = np.random.default_rng(3)
    old = rng.integers(0, 256, 1 << 20, dtype=np.uint8).tobytes()
    new = bytearray(old)
    for a in rng.choice((1 << 20) - 4, 100, replace=False):
        new[a:a + 4] = rng.integers(0, 256, 4, dtype=np.uint8).tobytes()
    new = bytes(new)
    p = transfer.create_patch(old, new)
    assert transfer.apply_patch(old, p) == new
    assert len(p) < 0.05 * len(new)


def test_large_device_buffers():
    """256 MB device buffers (a cfg4-style table slice) with scattered edits."""
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    old = torch.randint(0, 256, (256 << 20,), generator=g, device=dev, dtype=torch.uint8)
    new = old.clone()
    pos = torch.randint(0, (256 << 20) - 8, (20000,), generator=g, device=dev)
    new[pos] ^= 0x5A
    new[pos + 3] ^= 0x11
    p = transfer.create_patch(old, new)
    ops = fo.diff_ops(old.cpu().numpy().tobytes(), new.cpu().numpy().tobytes())
    assert len(ops) > 1000
    hn = new.cpu().numpy().tobytes()
    ref = b"".join(fo.encode_varint(a - (ops[i - 1][1] if i else 0)) + fo.encode_varint(b - a)
                   + hn[a:b] for i, (a, b) in enumerate(ops))
    assert p[32:] == ref
    assert transfer.apply_patch(old, p) == hn


def test_apply_errors():
    old, new = b"0123456789" * 10, b"0123456789" * 9 + b"abcdefghij"
    p = transfer.create_patch(old, new)
    with pytest.raises(StaleBaseError):
        transfer.apply_patch(old[:-1] + b"x", p)
    bad = bytearray(p)
    bad[-1] ^= 0xFF
    with pytest.raises(CorruptionError):
        transfer.apply_patch(old, bytes(bad))
    with pytest.raises(FormatError):
        transfer.apply_patch(old, p[:-3])  # truncated payload
    with pytest.raises(FormatError):
        transfer.apply_patch(old, p[:20])
    over = p[:32] + fo.encode_varint(95) + fo.encode_varint(50) + b"z" * 50
    with pytest.raises(FormatError):  # op past target_length
        transfer.apply_patch(old, over)


def test_quantized_update_pipeline():
    dev = torch.device("cuda:0")
    cfg = ModelConfig(n_fields=8, k=4, hidden_sizes=(16,), hash_bits=14)
    st = WeightStore(cfg, dev, with_optimizer=False)
    g = torch.Generator(device=dev).manual_seed(0)
    for _, t in st.blocks(False):
        t.view(-1).copy_(torch.randn(t.numel(), generator=g, device=dev) * 0.05)
    blob0 = transfer.quantized_blob(st)
    assert len(transfer.quantized_update_pipeline(blob0, st)) == 32  # unchanged round
    # one online round touching 1% of the weights
    n = st.ffm.numel()
    sel = torch.randperm(n, generator=g, device=dev)[: n // 100]
    st.ffm.view(-1)[sel] += torch.randn(sel.numel(), generator=g, device=dev) * 0.01
    blob1 = transfer.quantized_blob(st)
    p = transfer.quantized_update_pipeline(blob0, st)
    assert transfer.apply_patch(blob0, p) == blob1
    assert len(p) <= 0.15 * len(blob1)
