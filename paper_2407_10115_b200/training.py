"""Drop-in for ``fieldwise.training`` (T: training.py) on the GPU.

The reference's public loops keep their signatures and semantics:

* ``train_stream(source, store, schema, opts)`` -- the predict-then-learn
  schedule over text lines (T:172-218): blank lines skipped, unparseable lines
  counted and skipped, progressive logloss + 30k-window AUC, TrainAborted from
  the source carries the partial report.
* ``evaluate_stream(source, store, schema)`` -- score-only (T:221-236).
* ``hogwild_train(source, store, schema, opts)`` -- lock-free parallel mode
  (T:242-336) with ``opts.n_threads`` workers.

Underneath, lines are parsed in chunks by K10 (csrc/parse.cu), expanded to the
padded layout by K9, and trained by K2 -- the reference's exact sequential
schedule (forward -> record the progressive probability -> backward_update,
batch size 1) inside ONE persistent kernel per chunk (csrc/train.cu) -- or by
K6 (n_threads concurrent GPU workers sharing the store).  Metrics come from K8.
The batched array forms ``train_sequential`` / ``hogwild_train_arrays`` /
``evaluate_arrays`` take the padded device layout directly.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import (ContractError, FieldwiseError, HogwildWorkerError, NumericError,
                     TrainAborted)
from .features import InputSchema, pack_examples, parse_lines
from .metrics import StreamingEvaluator, stream_metrics_gpu, window_auc
from .model import WeightStore, _as_device, _status, predict_batch

DEFAULT_EVAL_WINDOW = 30000  # T:31
IPC_CHUNK_LINES = 256  # T:32 (the reference's worker feed granularity)
PARSE_CHUNK_LINES = 1 << 17  # lines parsed + trained per K10/K2 round


@dataclass
class TrainOptions:
    """T:35-46.  ``chunk`` (examples per K2 launch) is a GPU-side knob."""

    n_threads: int = 1
    prefetch_depth: int = 1
    eval_window: int = DEFAULT_EVAL_WINDOW
    sparse_updates: bool = True
    chunk: int = 1 << 20

    def __post_init__(self):
        if self.n_threads < 1:
            raise ContractError("n_threads must be >= 1")
        if self.prefetch_depth < 1:
            raise ContractError("prefetch_depth must be >= 1")


@dataclass
class TrainReport:
    """T:49-63 (+ ``probs``: every example's progressive prediction, f64)."""

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
    """The K2 train-state POD and scratch for one store and slot count M."""

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

    def _launch(self, fn, idx, val, labels, prob_out, *extra):
        st = _status(self.store.device)
        s = torch.cuda.current_stream(self.store.device)
        st.clear()
        rc = fn(self.store.c_model_ref(), ctypes.byref(self.ts), idx.data_ptr(), val.data_ptr(),
                labels.data_ptr(), self.M, idx.shape[0], *extra, prob_out.data_ptr(),
                self.scratch.data_ptr(), st.ptr(), s.cuda_stream)
        _lib.check(rc, fn.__name__)
        st.fetch_async()
        s.synchronize()
        return st

    def run(self, idx, val, labels, prob_out, base: int = 0):
        """K2 over one chunk; raises with the GLOBAL example number (base + i)."""
        self._launch(_lib.lib().dffm_train_sequential, idx, val, labels,
                     prob_out).raise_if_set("train: ", base)

    def run_hogwild(self, idx, val, labels, prob_out, n_workers: int, base: int = 0):
        self._launch(_lib.lib().dffm_train_hogwild, idx, val, labels, prob_out,
                     n_workers).raise_if_set("hogwild worker: ", base)


def _bump_on_failure(store: WeightStore, exc: Exception, c0: int):
    """Examples before the failing one were applied (one version bump each,
    M:532), so ForwardState / cache staleness checks stay exact."""
    ex = getattr(exc, "example", None)
    if ex is not None and ex >= c0:
        store.version += int(ex) - c0


def _report_gpu(dprobs, dlabels, window, start, probs, with_auc=True, parse_errors=0):
    if dprobs:
        series, loss_sum, count = stream_metrics_gpu(torch.cat(dprobs), torch.cat(dlabels), window)
    else:
        series, loss_sum, count = [], 0.0, 0
    wall = time.perf_counter() - start
    return TrainReport(examples_seen=count, parse_errors=parse_errors,
                       progressive_logloss=loss_sum / count if count else float("nan"),
                       rolling_auc_series=series if with_auc else [], wall_time=wall,
                       throughput=count / wall if wall > 0 else 0.0, probs=probs)


def _report(ev, start, probs, parse_errors=0):
    wall = time.perf_counter() - start
    return TrainReport(examples_seen=ev.count, parse_errors=parse_errors,
                       progressive_logloss=ev.mean_logloss, rolling_auc_series=ev.auc_series,
                       wall_time=wall, throughput=ev.count / wall if wall > 0 else 0.0,
                       probs=probs)


# ------------------------------------------------------------------ array forms


def train_sequential(idx, val, labels, store: WeightStore, opts: TrainOptions | None = None,
                     evaluator: StreamingEvaluator | None = None) -> TrainReport:
    """Predict-then-learn over padded arrays, in order (T:172-218 schedule).

    idx int32 [n,F,M], val f32 [n,F,M], labels uint8 [n] (host or device)."""
    opts = opts or TrainOptions()
    gpu_eval = evaluator is None  # K8 on the device stream unless the caller keeps state
    ev = evaluator or StreamingEvaluator(opts.eval_window)
    start = time.perf_counter()
    dev = store.device
    n = int(idx.shape[0])
    trainer = _Trainer(store, int(idx.shape[2]), opts.sparse_updates)
    probs = np.empty(n)
    dprobs, dlabels = [], []
    for c0 in range(0, n, opts.chunk):
        c1 = min(n, c0 + opts.chunk)
        ci = _as_device(idx[c0:c1], torch.int32, dev)
        cv = _as_device(val[c0:c1], torch.float32, dev)
        cl = _as_device(labels[c0:c1], torch.uint8, dev)
        po = torch.empty(c1 - c0, dtype=torch.float64, device=dev)
        try:
            trainer.run(ci, cv, cl, po, base=c0)
        except FieldwiseError as exc:
            _bump_on_failure(store, exc, c0)
            raise
        store.version += c1 - c0  # one bump per example (M:532)
        p = po.cpu().numpy()
        probs[c0:c1] = p
        if gpu_eval:
            dprobs.append(po)
            dlabels.append(cl)
        else:
            ev.add_batch(p, cl.cpu().numpy())
    if gpu_eval:
        return _report_gpu(dprobs, dlabels, opts.eval_window, start, probs)
    return _report(ev, start, probs)


def max_hogwild_workers(store: WeightStore, max_per_field: int) -> int:
    """Workers K6 can run concurrently on this GPU for this model shape."""
    return int(_lib.lib().dffm_hogwild_max_workers(store.c_model_ref(), max_per_field))


def hogwild_train_arrays(idx, val, labels, store: WeightStore, opts: TrainOptions | None = None
                         ) -> TrainReport:
    """Lock-free parallel single pass (T:269-336) over padded arrays.

    ``opts.n_threads`` workers run the predict-then-learn loop concurrently
    against the SHARED store with no locks (worker w takes examples w,
    w + n, ...); concurrent updates may overwrite each other (T:1-11).
    ``n_threads`` above what the GPU holds at once is capped to that number
    (``max_hogwild_workers``).  A failing worker stops the pool and surfaces
    as HogwildWorkerError with that worker's id."""
    opts = opts or TrainOptions()
    n_req = int(opts.n_threads)
    if n_req == 1:
        try:
            return train_sequential(idx, val, labels, store, opts)
        except FieldwiseError as exc:
            raise HogwildWorkerError(f"worker 0 failed: {exc}", worker_id=0) from exc
    start = time.perf_counter()
    dev = store.device
    n = int(idx.shape[0])
    M = int(idx.shape[2])
    trainer = _Trainer(store, M, opts.sparse_updates)
    n_workers = max(1, min(n_req, max_hogwild_workers(store, M)))
    probs = np.empty(n)
    dprobs, dlabels = [], []
    for c0 in range(0, n, opts.chunk):
        c1 = min(n, c0 + opts.chunk)
        ci = _as_device(idx[c0:c1], torch.int32, dev)
        cv = _as_device(val[c0:c1], torch.float32, dev)
        cl = _as_device(labels[c0:c1], torch.uint8, dev)
        po = torch.empty(c1 - c0, dtype=torch.float64, device=dev)
        try:
            trainer.run_hogwild(ci, cv, cl, po, n_workers, base=c0)
        except FieldwiseError as exc:
            store.mark_mutated()  # T:318: the workers' own bumps are not visible
            ex = getattr(exc, "example", None)
            wid = (int(ex) - c0) % n_workers if ex is not None else -1
            raise HogwildWorkerError(f"worker {wid} failed: {exc}", worker_id=wid) from exc
        probs[c0:c1] = po.cpu().numpy()
        dprobs.append(po)
        dlabels.append(cl)
    store.mark_mutated()  # T:318
    return _report_gpu(dprobs, dlabels, opts.eval_window, start, probs, with_auc=False)


def evaluate_arrays(idx, val, labels, store: WeightStore):
    """Score without updating -> (auc, logloss, n) over padded arrays (T:221-236)."""
    n = int(idx.shape[0])
    if n == 0:
        return None, float("nan"), 0
    p = predict_batch(idx, val, store).double().cpu().numpy()
    y = np.asarray(labels.cpu() if isinstance(labels, torch.Tensor) else labels).astype(np.int64)
    losses = np.where(y == 1, -np.log(p), -np.log1p(-p))
    return window_auc(p, y), float(losses.mean()), n


# ------------------------------------------------------------------ text sources


def _line_bytes(line) -> bytes:
    b = line if isinstance(line, (bytes, bytearray)) else str(line).encode("utf-8")
    return bytes(b).rstrip(b"\n") + b"\n"


def _chunks(source, n_lines: int):
    """Lists of at most n_lines lines; a TrainAborted raised by the source is
    re-raised after the lines read before it are handed out (the reference has
    trained every line it read when the source fails)."""
    buf = []
    it = iter(source)
    while True:
        try:
            line = next(it)
        except StopIteration:
            break
        except TrainAborted:
            if buf:
                yield buf
            raise
        buf.append(line)
        if len(buf) >= n_lines:
            yield buf
            buf = []
    if buf:
        yield buf


def _unpack_rows(parsed, keep: torch.Tensor):
    """K9: parsed ragged lines -> padded idx/val [n, F, M] on the device, rows
    restricted to ``keep`` (lines that parsed), in stream order."""
    b = parsed.batch
    n, F, M = b.n, b.n_fields, b.max_per_field
    dev = b.cnt.device
    pi = torch.empty((n, F, M), dtype=torch.int32, device=dev)
    pv = torch.empty((n, F, M), dtype=torch.float32, device=dev)
    st = _status(dev)
    st.clear()
    if n:
        _lib.check(_lib.lib().dffm_unpack_ragged(
            b.ex_off.data_ptr(), b.cnt.data_ptr(), b.idx.data_ptr(), b.val.data_ptr(), n, F, M,
            0, pi.data_ptr(), pv.data_ptr(), 0, st.ptr(),
            torch.cuda.current_stream(dev).cuda_stream), "dffm_unpack_ragged")
    return pi[keep], pv[keep], parsed.labels[keep]


def _parse_chunk(lines, schema: InputSchema, device, strict: bool):
    """K10 over a chunk of lines -> (idx, val, labels, parse_errors) of the
    lines that parsed, blank lines dropped (T:176).  ``strict`` raises
    ParseError at the first bad line (evaluate_stream, T:228); otherwise bad
    lines are counted and skipped (train_stream, T:178-181).  Lines the
    reference accepts but K10 cannot take (non-ASCII whitespace or digits,
    > 1024 features, > 255 in one field) raise ContractError either way."""
    from .errors import ParseError
    from .features import PARSE_ERRORS
    text = b"".join(_line_bytes(ln) for ln in lines)
    parsed = parse_lines(text, schema, device, raise_on_error=False, skip_blank=True)
    status = parsed.status
    unsupported = torch.nonzero((status >= 8) & (status <= 10))
    bad = torch.nonzero((status != 0) & (status != 11))
    if unsupported.numel():
        i = int(unsupported[0, 0])
        raise ContractError(f"line {i + 1} of the chunk: "
                            f"{PARSE_ERRORS[int(status[i])]}")
    if strict and bad.numel():
        i = int(bad[0, 0])
        raise ParseError(f"line {i + 1} of the chunk: "
                         f"{PARSE_ERRORS.get(int(status[i]), 'parse error')}")
    keep = status == 0
    idx, val, labels = _unpack_rows(parsed, keep)
    return idx, val, labels, int(bad.shape[0])


def train_stream(source, store: WeightStore, schema: InputSchema,
                 opts: TrainOptions | None = None) -> TrainReport:
    """Train on a line source in order: score first, learn second (T:188-218).

    Progressive validation: no example influences its own prediction.
    Unparseable lines are counted and skipped; an I/O failure (TrainAborted
    from the source) aborts with the partial report attached."""
    return _train_text(source, store, schema, opts or TrainOptions(), hogwild=False)


def hogwild_train(source, store: WeightStore, schema: InputSchema,
                  opts: TrainOptions | None = None) -> TrainReport:
    """Parallel single pass with lock-free shared-weight updates (T:269-336):
    ``opts.n_threads`` K6 workers; the rolling AUC series is reported only for
    one worker, where the run is the sequential schedule byte for byte."""
    return _train_text(source, store, schema, opts or TrainOptions(), hogwild=True)


def _train_text(source, store, schema, opts, hogwild: bool) -> TrainReport:
    if schema.n_fields != store.config.n_fields or schema.hash_bits != store.config.hash_bits:
        raise ContractError("schema does not match the model (fields / hash_bits)")
    start = time.perf_counter()
    dev = store.device
    parse_errors = 0
    dprobs, dlabels, probs = [], [], []
    trainers = {}
    seen = 0
    n_workers = int(opts.n_threads)

    def report():
        p = np.concatenate(probs) if probs else np.empty(0)
        return _report_gpu(dprobs, dlabels, opts.eval_window, start, p,
                           with_auc=not hogwild or n_workers == 1, parse_errors=parse_errors)

    try:
        for lines in _chunks(source, PARSE_CHUNK_LINES):
            idx, val, labels, nbad = _parse_chunk(lines, schema, dev, strict=False)
            parse_errors += nbad
            n = int(idx.shape[0])
            if n == 0:
                continue
            M = int(idx.shape[2])
            if M not in trainers:
                trainers[M] = _Trainer(store, M, opts.sparse_updates)
            tr = trainers[M]
            po = torch.empty(n, dtype=torch.float64, device=dev)
            if hogwild:
                # the reference's workers bump their own (forked) copies of the
                # version; the caller's store is marked mutated once (T:318)
                w = max(1, min(n_workers, max_hogwild_workers(store, M)))
                try:
                    if w == 1:
                        tr.run(idx, val, labels, po, base=seen)
                    else:
                        tr.run_hogwild(idx, val, labels, po, w, base=seen)
                except FieldwiseError as exc:
                    store.mark_mutated()
                    ex = getattr(exc, "example", None)
                    wid = (int(ex) - seen) % w if ex is not None else -1
                    raise HogwildWorkerError(f"worker {wid} failed: {exc}",
                                             worker_id=wid) from exc
            else:
                try:
                    tr.run(idx, val, labels, po, base=seen)
                except FieldwiseError as exc:
                    _bump_on_failure(store, exc, seen)
                    raise
                store.version += n  # M:532, one bump per example
            seen += n
            dprobs.append(po)
            dlabels.append(labels)
            probs.append(po.cpu().numpy())
    except TrainAborted as exc:
        exc.partial_report = report()
        raise
    if hogwild:
        store.mark_mutated()  # T:318
    return report()


def evaluate_stream(source, store: WeightStore, schema: InputSchema):
    """Score a labeled stream without updating; returns (auc, logloss, n)
    (T:221-236).  Every non-blank line must parse (ParseError otherwise)."""
    if schema.n_fields != store.config.n_fields or schema.hash_bits != store.config.hash_bits:
        raise ContractError("schema does not match the model (fields / hash_bits)")
    dev = store.device
    scores, labels_all = [], []
    for lines in _chunks(source, PARSE_CHUNK_LINES):
        idx, val, labels, _ = _parse_chunk(lines, schema, dev, strict=True)
        if idx.shape[0]:
            scores.append(predict_batch(idx, val, store).double().cpu().numpy())
            labels_all.append(labels.cpu().numpy())
    if not scores:
        return None, float("nan"), 0
    p = np.concatenate(scores)
    y = np.concatenate(labels_all).astype(np.int64)
    loss_sum = 0.0
    for v in np.where(y == 1, -np.log(p), -np.log1p(-p)).tolist():  # T:233, in order
        loss_sum += v
    return window_auc(p, y), loss_sum / len(p), len(p)


# ------------------------------------------------------------------ one example


def _train_one(example, label: int, store: WeightStore, sparse: bool) -> float:
    """K2 on one ParsedExample-like object (model.backward_update's engine);
    returns the clamped progressive probability (the loss's p, M:460)."""
    idx, val, _ = pack_examples([example], store.config.n_fields)
    lab = np.array([label], np.uint8)
    rep = train_sequential(idx, val, lab, store, TrainOptions(sparse_updates=sparse))
    return float(rep.probs[0])


def backward_update(state, example, label: int, store: WeightStore, sparse: bool = True) -> float:
    """Re-export of model.backward_update (M:440) for callers of the old path."""
    from .model import backward_update as bu
    return bu(state, example, label, store, sparse)
