"""Drop-in for ``fieldwise.training`` (T: training.py) on the GPU.

``train_sequential`` runs the reference's predict-then-learn schedule
(T:172-185: forward -> record the progressive probability -> backward_update,
example by example, batch size 1) inside ONE persistent kernel (K2,
csrc/train.cu) over a resident batch of examples; the host only feeds chunks
and folds the returned probabilities into the progressive metrics.
``evaluate_stream`` is the score-only loop (T:221-236) over K1.
``hogwild_train`` is the lock-free parallel mode (T:242-336) as K6: n_threads
concurrent GPU workers sharing the store.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ContractError, FieldwiseError, HogwildWorkerError, TrainAborted
from .features import pack_examples
from .metrics import StreamingEvaluator, stream_metrics_gpu, window_auc
from .model import WeightStore, _as_device, _status, predict_batch

DEFAULT_EVAL_WINDOW = 30000  # T:31


@dataclass
class TrainOptions:
    """T:35-46 (n_threads / prefetch_depth are accepted for API parity; the
    GPU schedule is a single in-order stream)."""

    n_threads: int = 1
    prefetch_depth: int = 1
    eval_window: int = DEFAULT_EVAL_WINDOW
    sparse_updates: bool = True
    chunk: int = 1 << 20  # examples staged per K2 launch

    def __post_init__(self):
        if self.n_threads < 1:
            raise ContractError("n_threads must be >= 1")
        if self.prefetch_depth < 1:
            raise ContractError("prefetch_depth must be >= 1")


@dataclass
class TrainReport:
    """T:49-63."""

    examples_seen: int = 0
    parse_errors: int = 0
    progressive_logloss: float = float("nan")
    rolling_auc_series: list = field(default_factory=list)
    wall_time: float = 0.0
    throughput: float = 0.0
    probs: np.ndarray | None = None

    def summary(self) -> str:
        return (f"examples={self.examples_seen} parse_errors={self.parse_errors}"
                f" logloss={self.progressive_logloss:.6f}"
                f" wall={self.wall_time:.2f}s throughput={self.throughput:.0f}/s")


class _Trainer:
    """Holds the K2 train-state POD and scratch for one store."""

    def __init__(self, store: WeightStore, max_per_field: int, sparse: bool):
        if store.wdtype != "f32" or not store.has_optimizer:
            raise ContractError("training needs an f32 store with optimizer state")
        self.store = store
        cfg = store.config
        ts = _lib.DffmTrainState()
        ts.lr_acc = store.lr_acc.data_ptr()
        ts.ffm_acc = store.ffm_acc.data_ptr()
        for i, (w, b) in enumerate(store.nn_accs):
            ts.W_acc[i] = w.data_ptr()
            ts.b_acc[i] = b.data_ptr()
        ts.lr_ffm, ts.lr_lr, ts.lr_nn, ts.power_t = cfg.lr_ffm, cfg.lr_lr, cfg.lr_nn, cfg.power_t
        ts.sparse = 1 if sparse else 0
        self.ts = ts
        self.M = max_per_field
        nbytes = int(_lib.lib().dffm_train_scratch_bytes(store.c_model_ref(), max_per_field))
        self.scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=store.device)

    def run_hogwild(self, idx, val, labels, prob_out, n_workers: int):
        import ctypes
        st = _status(self.store.device)
        s = torch.cuda.current_stream(self.store.device)
        st.clear()
        rc = _lib.lib().dffm_train_hogwild(
            self.store.c_model_ref(), ctypes.byref(self.ts), idx.data_ptr(), val.data_ptr(),
            labels.data_ptr(), self.M, idx.shape[0], n_workers, prob_out.data_ptr(),
            self.scratch.data_ptr(), st.ptr(), s.cuda_stream)
        _lib.check(rc, "dffm_train_hogwild")
        st.fetch_async()
        s.synchronize()
        st.raise_if_set("hogwild worker: ")

    def run(self, idx: torch.Tensor, val: torch.Tensor, labels: torch.Tensor,
            prob_out: torch.Tensor, check=True):
        import ctypes
        st = _status(self.store.device)
        s = torch.cuda.current_stream(self.store.device)
        st.clear()
        n = idx.shape[0]
        rc = _lib.lib().dffm_train_sequential(
            self.store.c_model_ref(), ctypes.byref(self.ts), idx.data_ptr(), val.data_ptr(),
            labels.data_ptr(), self.M, n, prob_out.data_ptr(), self.scratch.data_ptr(),
            st.ptr(), s.cuda_stream)
        _lib.check(rc, "dffm_train_sequential")
        if check:
            st.fetch_async()
            s.synchronize()
            st.raise_if_set("train: ")


def train_sequential(idx, val, labels, store: WeightStore, opts: TrainOptions | None = None,
                     evaluator: StreamingEvaluator | None = None) -> TrainReport:
    """Predict-then-learn over padded arrays, in order (T:172-218).

    idx int32 [n,F,M], val f32 [n,F,M], labels uint8 [n] (host or device)."""
    opts = opts or TrainOptions()
    gpu_eval = evaluator is None  # K8 on the device stream unless the caller keeps state
    ev = evaluator or StreamingEvaluator(opts.eval_window)
    start = time.perf_counter()
    dev = store.device
    n = int(idx.shape[0])
    M = int(idx.shape[2])
    trainer = _Trainer(store, M, opts.sparse_updates)
    probs = np.empty(n)
    dprobs, dlabels = [], []
    for c0 in range(0, n, opts.chunk):
        c1 = min(n, c0 + opts.chunk)
        ci = _as_device(idx[c0:c1], torch.int32, dev)
        cv = _as_device(val[c0:c1], torch.float32, dev)
        cl = _as_device(labels[c0:c1], torch.uint8, dev)
        po = torch.empty(c1 - c0, dtype=torch.float64, device=dev)
        try:
            trainer.run(ci, cv, cl, po)
        except Exception as exc:
            rep = _report(ev, start, probs[:c0])
            if isinstance(exc, (TrainAborted,)):
                exc.partial_report = rep
            raise
        store.version += c1 - c0  # one bump per example (M:532)
        p = po.cpu().numpy()
        probs[c0:c1] = p
        if gpu_eval:
            dprobs.append(po)
            dlabels.append(cl)
        else:
            ev.add_batch(p, np.asarray(labels[c0:c1].cpu() if isinstance(labels, torch.Tensor)
                                       else labels[c0:c1]))
    if gpu_eval:
        return _report_gpu(dprobs, dlabels, opts.eval_window, start, probs)
    return _report(ev, start, probs)


def _report_gpu(dprobs, dlabels, window, start, probs, with_auc=True):
    if dprobs:
        series, loss_sum, count = stream_metrics_gpu(torch.cat(dprobs), torch.cat(dlabels), window)
    else:
        series, loss_sum, count = [], 0.0, 0
    wall = time.perf_counter() - start
    return TrainReport(examples_seen=count,
                       progressive_logloss=loss_sum / count if count else float("nan"),
                       rolling_auc_series=series if with_auc else [], wall_time=wall,
                       throughput=count / wall if wall > 0 else 0.0, probs=probs)


def _report(ev, start, probs):
    wall = time.perf_counter() - start
    return TrainReport(examples_seen=ev.count, progressive_logloss=ev.mean_logloss,
                       rolling_auc_series=ev.auc_series, wall_time=wall,
                       throughput=ev.count / wall if wall > 0 else 0.0, probs=probs)


def train_stream(examples, store: WeightStore, opts: TrainOptions | None = None) -> TrainReport:
    """train_stream over ParsedExample-like objects (T:188-218)."""
    idx, val, labels = pack_examples(list(examples), store.config.n_fields)
    return train_sequential(idx, val, labels, store, opts)


def max_hogwild_workers(store: WeightStore, max_per_field: int) -> int:
    """Workers K6 can run concurrently on this GPU for this model shape."""
    return int(_lib.lib().dffm_hogwild_max_workers(store.c_model_ref(), max_per_field))


def hogwild_train(idx, val, labels, store: WeightStore, opts: TrainOptions | None = None
                  ) -> TrainReport:
    """Lock-free parallel single pass (T:269-336) over padded arrays.

    ``opts.n_threads`` workers run the predict-then-learn loop concurrently
    against the SHARED store with no locks (worker w takes examples w,
    w + n, ...); concurrent updates may overwrite each other (T:1-11).
    Progressive metrics are computed over every example's pre-update
    prediction; the rolling AUC series is reported only for one worker, where
    the run is the sequential schedule itself (identical to train_stream).
    A failing worker stops the pool and surfaces as HogwildWorkerError."""
    opts = opts or TrainOptions()
    n_workers = int(opts.n_threads)
    if n_workers == 1:
        try:
            return train_sequential(idx, val, labels, store, opts)
        except FieldwiseError as exc:
            raise HogwildWorkerError(f"worker 0 failed: {exc}", worker_id=0) from exc
    start = time.perf_counter()
    dev = store.device
    n = int(idx.shape[0])
    M = int(idx.shape[2])
    trainer = _Trainer(store, M, opts.sparse_updates)
    probs = np.empty(n)
    dprobs, dlabels = [], []
    for c0 in range(0, n, opts.chunk):
        c1 = min(n, c0 + opts.chunk)
        ci = _as_device(idx[c0:c1], torch.int32, dev)
        cv = _as_device(val[c0:c1], torch.float32, dev)
        cl = _as_device(labels[c0:c1], torch.uint8, dev)
        po = torch.empty(c1 - c0, dtype=torch.float64, device=dev)
        try:
            trainer.run_hogwild(ci, cv, cl, po, n_workers)
        except FieldwiseError as exc:
            store.mark_mutated()  # T:318: the workers' own bumps are not visible
            ex = getattr(exc, "example", None)
            wid = int(ex) % n_workers if ex is not None else -1
            raise HogwildWorkerError(f"worker {wid} failed: {exc}", worker_id=wid) from exc
        probs[c0:c1] = po.cpu().numpy()
        dprobs.append(po)
        dlabels.append(cl)
    store.mark_mutated()  # T:318
    return _report_gpu(dprobs, dlabels, opts.eval_window, start, probs, with_auc=False)


def backward_update(state, example, label: int, store: WeightStore, sparse: bool = True) -> float:
    """Single-example learn step with the reference's contract (M:440-533).

    K2 recomputes the forward pass inside the fused step (identical to
    ``state``), applies the Adagrad updates and returns the log-loss."""
    if getattr(state, "_store", None) is not store or state._store_version != store.version:
        raise ContractError("forward state was not produced against this store state")
    if label not in (0, 1):
        raise ContractError(f"label must be 0 or 1, got {label!r}")
    idx, val, _ = pack_examples([example], store.config.n_fields)
    lab = np.array([label], np.uint8)
    rep = train_sequential(idx, val, lab, store, TrainOptions(sparse_updates=sparse))
    p = float(rep.probs[0])
    return -math.log(p) if label else -math.log1p(-p)


def evaluate_stream(idx, val, labels, store: WeightStore):
    """Score without updating -> (auc, logloss, n) (T:221-236)."""
    n = int(idx.shape[0])
    if n == 0:
        return None, float("nan"), 0
    p = predict_batch(idx, val, store).double().cpu().numpy()
    y = np.asarray(labels.cpu() if isinstance(labels, torch.Tensor) else labels).astype(np.int64)
    losses = np.where(y == 1, -np.log(p), -np.log1p(-p))
    return window_auc(p, y), float(losses.mean()), n
