"""K6 Hogwild-style trainer (T:242-336) against its SPEC contract:
N=1 is the sequential schedule exactly; N>1 workers share the store with no
locks and must land within 2% relative progressive logloss of the N=1 run;
a failing worker surfaces as HogwildWorkerError; N workers beat N=1 on
throughput."""

import numpy as np
import pytest
import torch

from paper_2407_10115_b200 import configs, synth
from paper_2407_10115_b200.errors import ContractError, HogwildWorkerError
from paper_2407_10115_b200.model import ModelConfig, WeightStore, predict_batch
from paper_2407_10115_b200.training import (TrainOptions, hogwild_train_arrays, max_hogwild_workers,
                                             train_sequential)

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
BITS = 14


def make_store(seed=3):
    cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=BITS, lr_ffm=0.05,
                      lr_lr=0.05, lr_nn=0.05)
    st = WeightStore(cfg, DEV).fill_accumulators(1.0)
    g = torch.Generator(device=DEV).manual_seed(seed)
    for t in [st.lr, st.ffm] + [x for wb in st.nn_layers for x in wb]:
        t.view(-1).copy_(torch.randn(t.numel(), generator=g, device=DEV) * 0.05)
    return st


def planted_stream(n, seed=11):
    """cfg3 schema at 2^14 buckets; labels ~ Bernoulli(teacher DeepFFM)."""
    idx, val = synth.make_examples(configs.CFG3, n, seed=seed, hash_bits=BITS, device=DEV)
    teacher = make_store(seed=99)
    p = predict_batch(idx, val, teacher)
    g = torch.Generator(device=DEV).manual_seed(seed + 1)
    labels = (torch.rand(n, generator=g, device=DEV) < p).to(torch.uint8)
    return idx, val, labels


def snapshot(st):
    return [t.detach().clone() for _, t in st.blocks(True)]


def test_one_worker_is_the_sequential_schedule():
    idx, val, labels = planted_stream(3000)
    a, b = make_store(), make_store()
    ra = hogwild_train_arrays(idx, val, labels, a, TrainOptions(n_threads=1))
    rb = train_sequential(idx, val, labels, b, TrainOptions())
    for x, y in zip(snapshot(a), snapshot(b)):
        assert torch.equal(x, y)  # byte-identical weights and accumulators
    assert np.array_equal(ra.probs, rb.probs)
    assert ra.rolling_auc_series == rb.rolling_auc_series


def test_parallel_workers_logloss_within_two_percent():
    n = 40000
    idx, val, labels = planted_stream(n)
    ref = hogwild_train_arrays(idx, val, labels, make_store(), TrainOptions(n_threads=1))
    for w in (4, 32):
        st = make_store()
        v0 = st.version
        rep = hogwild_train_arrays(idx, val, labels, st, TrainOptions(n_threads=w))
        assert rep.examples_seen == n and np.isfinite(rep.progressive_logloss)
        assert rep.rolling_auc_series == []  # only meaningful for one worker
        assert st.version == v0 + 1          # T:318 mark_mutated
        rel = abs(rep.progressive_logloss - ref.progressive_logloss) / ref.progressive_logloss
        assert rel < 0.02, (w, rep.progressive_logloss, ref.progressive_logloss)
        # every weight stays finite and every example got a probability
        assert np.all((rep.probs > 0) & (rep.probs < 1))
        for _, t in st.blocks(True):
            assert torch.isfinite(t).all()


def test_worker_failure_surfaces_with_worker_id():
    idx, val, labels = planted_stream(2000)
    labels = labels.clone()
    labels[777] = 2  # M:453-454 ContractError inside a worker
    w = 8
    with pytest.raises(HogwildWorkerError) as ei:
        hogwild_train_arrays(idx, val, labels, make_store(), TrainOptions(n_threads=w))
    assert ei.value.worker_id == 777 % w
    assert isinstance(ei.value.__cause__, ContractError)


def test_workers_scale_throughput():
    n = 20000
    idx, val, labels = planted_stream(n)
    hogwild_train_arrays(idx[:500], val[:500], labels[:500], make_store(), TrainOptions(n_threads=64))
    r1 = hogwild_train_arrays(idx, val, labels, make_store(), TrainOptions(n_threads=1))
    w = min(64, max_hogwild_workers(make_store(), idx.shape[2]))
    rw = hogwild_train_arrays(idx, val, labels, make_store(), TrainOptions(n_threads=w))
    assert rw.throughput >= 2 * r1.throughput, (rw.throughput, r1.throughput)
