"""Streaming evaluation (Me: /root/reference/pkg/src/fieldwise/metrics.py).

Host-side restatement of the reference's progressive logloss, 30k
non-overlapping-window midrank AUC and RIG (Me:21-139), fed with the
probabilities the GPU kernels return.  Vectorised numpy: a whole window (or a
whole progressive stream) is folded at once instead of one Python call per
example.  Checked against the reference's own outputs (golden metrics.npz) in
tests/test_host.py and, for the K8 device evaluator, tests/test_gpu_eval.py.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ContractError

LOSS_CLAMP = 1e-7  # Me:18


def _midranks(x: np.ndarray) -> np.ndarray:
    """1-based ranks with ties averaged (scipy.stats.rankdata 'average')."""
    order = np.argsort(x, kind="mergesort")
    xs = x[order]
    n = len(x)
    starts = np.flatnonzero(np.r_[True, xs[1:] != xs[:-1]])
    ends = np.r_[starts[1:], n]
    avg = (starts + ends + 1) / 2.0
    r = np.empty(n)
    r[order] = np.repeat(avg, ends - starts)
    return r


def window_auc(scores, labels):
    """Mann-Whitney AUC with midranks; None for a single-class window (Me:21-34)."""
    labels = np.asarray(labels)
    n_pos = int(labels.sum())
    n_neg = len(labels) - n_pos
    if n_pos == 0 or n_neg == 0:
        return None
    ranks = _midranks(np.asarray(scores, dtype=np.float64))
    pos_rank_sum = float(ranks[labels == 1].sum())
    return (pos_rank_sum - n_pos * (n_pos + 1) / 2.0) / (n_pos * n_neg)


def _losses(p: np.ndarray, y: np.ndarray) -> np.ndarray:
    p = np.clip(np.asarray(p, np.float64), LOSS_CLAMP, 1.0 - LOSS_CLAMP)
    y = np.asarray(y)
    return np.where(y == 1, -np.log(p), -np.log1p(-p))


def logloss(pairs) -> float:
    """Mean NLL with clamped scores (Me:37-47)."""
    pairs = list(pairs)
    if not pairs:
        raise ContractError("logloss of an empty stream is undefined")
    p, y = zip(*pairs)
    return float(_losses(np.array(p), np.array(y)).mean())


def rig(pairs) -> float:
    """1 - logloss / H(base rate) (Me:50-59)."""
    pairs = list(pairs)
    if not pairs:
        raise ContractError("rig of an empty stream is undefined")
    q = sum(y for _, y in pairs) / len(pairs)
    if q in (0.0, 1.0):
        raise ContractError("rig needs both classes present")
    entropy = -(q * math.log(q) + (1.0 - q) * math.log(1.0 - q))
    return 1.0 - logloss(pairs) / entropy


def stream_metrics_gpu(probs, labels, window: int = 30000):
    """K8 (csrc/eval.cu): the StreamingEvaluator result for a whole device
    stream -> (auc_series [(count, auc | None)], loss_sum, count).  AUC is the
    exact Mann-Whitney count per window (same value as the midrank formula);
    per-window loss sums are folded in stream order on the host."""
    import torch

    from . import _lib
    if window < 2:
        raise ContractError("window capacity must be >= 2")
    p = probs.detach().reshape(-1).to(torch.float64).contiguous()
    y = labels.detach().reshape(-1).to(device=p.device, dtype=torch.uint8).contiguous()
    n = p.numel()
    if n == 0:
        return [], 0.0, 0
    n_full, n_win = n // window, -(-n // window)
    auc = torch.empty(max(n_full, 1), dtype=torch.float64, device=p.device)
    loss = torch.empty(n_win, dtype=torch.float64, device=p.device)
    _lib.check(_lib.lib().fw_eval_stream(p.data_ptr(), y.data_ptr(), n, window, auc.data_ptr(),
                                         loss.data_ptr(),
                                         torch.cuda.current_stream(p.device).cuda_stream),
               "fw_eval_stream")
    a = auc.cpu().numpy()[:n_full]
    series = [((i + 1) * window, None if math.isnan(v) else float(v)) for i, v in enumerate(a)]
    total = 0.0
    for v in loss.cpu().numpy().tolist():
        total += v
    return series, total, n


class MetricWindow:
    """Bounded buffer of recent (score, label) pairs (Me:62-90)."""

    def __init__(self, capacity: int = 30000):
        if capacity < 2:
            raise ContractError("window capacity must be >= 2")
        self.capacity = capacity
        self._scores: list = []
        self._labels: list = []

    def __len__(self) -> int:
        return len(self._scores)

    @property
    def full(self) -> bool:
        return len(self._scores) >= self.capacity

    def add(self, score: float, label: int):
        self._scores.append(score)
        self._labels.append(label)

    def auc(self):
        if not self._scores:
            return None
        return window_auc(self._scores, self._labels)

    def clear(self):
        self._scores.clear()
        self._labels.clear()


def rolling_auc(pairs, window: int = 30000):
    """Yield (examples_seen, auc_or_None) per completed non-overlapping window
    (Me:93-106)."""
    buf = MetricWindow(window)
    seen = 0
    for score, label in pairs:
        buf.add(score, label)
        seen += 1
        if buf.full:
            yield seen, buf.auc()
            buf.clear()


class StreamingEvaluator:
    """Progressive-validation accumulator (Me:109-129), batch-fed.

    ``add_batch(p, y)`` is equivalent to calling the reference's ``add`` per
    element in order: the log-loss sum accumulates sequentially (same f64
    additions, in order) and AUC windows close every ``window`` examples."""

    def __init__(self, window: int = 30000):
        if window < 2:
            raise ContractError("window capacity must be >= 2")
        self.window = window
        self.auc_series: list = []
        self.count = 0
        self.loss_sum = 0.0
        self._buf_p: list = []
        self._buf_y: list = []
        self._buf_n = 0

    def add(self, score: float, label: int):
        self.add_batch(np.array([score]), np.array([label]))

    def add_batch(self, scores, labels):
        p = np.asarray(scores, np.float64)
        y = np.asarray(labels).astype(np.int64)
        for v in _losses(p, y).tolist():  # strictly sequential f64 sum (Me:120)
            self.loss_sum += v
        i = 0
        n = len(p)
        while i < n:
            take = min(n - i, self.window - self._buf_n)
            self._buf_p.append(p[i:i + take])
            self._buf_y.append(y[i:i + take])
            self._buf_n += take
            self.count += take
            i += take
            if self._buf_n >= self.window:
                self.auc_series.append((self.count, window_auc(np.concatenate(self._buf_p),
                                                               np.concatenate(self._buf_y))))
                self._buf_p, self._buf_y, self._buf_n = [], [], 0

    @property
    def mean_logloss(self) -> float:
        return self.loss_sum / self.count if self.count else float("nan")


def format_metric_lines(series, final: dict, count: int):
    """Tab-separated metric stream (Me:132-139)."""
    lines = []
    for idx, auc in series:
        lines.append(f"{idx}\tauc\t{auc:.6f}" if auc is not None else f"{idx}\tauc\tnan")
    for name, value in final.items():
        lines.append(f"{count}\t{name}\t{value:.6f}")
    return lines
