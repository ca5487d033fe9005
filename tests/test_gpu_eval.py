"""K8 streaming evaluator (Me:21-34, Me:109-129) on the device vs the
reference's own metric outputs (tests/golden/metrics.npz) and the host
evaluator, including ties, one-class windows and a trailing partial window."""

import math

import numpy as np
import pytest
import torch

from paper_2407_10115_b200 import metrics
from tests.golden_io import load

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def gpu(p, y, w):
    return metrics.stream_metrics_gpu(torch.as_tensor(p, device=DEV),
                                      torch.as_tensor(np.asarray(y), device=DEV), w)


def test_matches_reference_golden():
    g = load("metrics")
    series, loss_sum, n = gpu(g["scores"], g["labels"], 30000)
    ref = [(int(c), float(a)) for c, a in g["series"]]
    assert [c for c, _ in series] == [c for c, _ in ref]
    for (_, a), (_, b) in zip(series, ref):
        assert a == pytest.approx(b, rel=1e-12)
    assert loss_sum / n == pytest.approx(float(g["mean_logloss"]), rel=1e-12)


@pytest.mark.parametrize("w", [2, 7, 1000, 30000])
def test_matches_host_evaluator_with_ties_and_degenerate_windows(w):
    rng = np.random.default_rng(w)
    n = 3 * w + w // 2 + 1
    p = np.round(rng.random(n), 2)                       # many ties
    p[: w // 3] = 0.5                                    # a tie-heavy prefix
    y = (rng.random(n) < 0.3).astype(np.int64)
    y[w:2 * w] = 1                                       # a one-class window -> None
    p[2 * w:3 * w] = 0.25                                # an all-ties window -> 0.5
    y[2 * w], y[2 * w + 1] = 0, 1
    ev = metrics.StreamingEvaluator(w)
    ev.add_batch(p, y)
    series, loss_sum, cnt = gpu(p, y, w)
    assert cnt == ev.count
    assert len(series) == len(ev.auc_series)
    for (c1, a1), (c2, a2) in zip(series, ev.auc_series):
        assert c1 == c2
        assert (a1 is None) == (a2 is None)
        if a1 is not None:
            assert a1 == pytest.approx(a2, rel=1e-12, abs=1e-15)
    assert series[1][1] is None
    assert series[2][1] == 0.5
    assert loss_sum == pytest.approx(ev.loss_sum, rel=1e-12)


def test_large_stream_and_empty():
    assert gpu(np.zeros(0), np.zeros(0, np.int64), 30000) == ([], 0.0, 0)
    rng = np.random.default_rng(0)
    n = 10_000_000  # a cfg3-length stream: 333 windows
    p = rng.random(n)
    y = (rng.random(n) < p).astype(np.uint8)
    series, loss_sum, cnt = gpu(p, y, 30000)
    assert cnt == n and len(series) == n // 30000
    ev = metrics.StreamingEvaluator(30000)
    ev.add_batch(p[:90000], y[:90000])
    for (c1, a1), (c2, a2) in zip(series[:3], ev.auc_series):
        assert c1 == c2 and a1 == pytest.approx(a2, rel=1e-12)
    assert all(0.6 < a < 0.9 for _, a in series)
    assert math.isfinite(loss_sum)
