"""Drop-in for ``fieldwise.model`` (M: /root/reference/pkg/src/fieldwise/model.py).

Same names and semantics -- ``ModelConfig``, ``WeightStore``, ``init_model``,
``forward``, ``predict_proba``, ``backward_update``, ``flat_weight_view``,
``store_from_bytes``, ``save_model``, ``load_model`` -- plus the batched
entry points the GPU makes worthwhile (``predict_batch``).

The store lives in HBM as separate, 256-byte-aligned blocks (torch tensors used
purely as device buffers) laid out exactly like the reference's frozen flat
array, block by block (M:145-153):

    lr   [2^b + 1]            f32 | bf16 | u16 (bias at 2^b)
    ffm  [2^b, F, k]          f32 | bf16 | u16   (row = one bucket's F*k latent
                                                  values: every field-aware
                                                  k-segment is a 16 B-aligned
                                                  vector load)
    W[l] [in, out] f32, b[l] [out] f32
    accumulators: same shapes, f32 (only when the store trains)

``flat_weight_view`` reassembles the reference byte layout on the host, so a
model file written here is byte-identical to one written by the reference.
Compute runs through libdffm.so (``_lib``); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ContractError, FormatError, NumericError, SizingError

MERGE_EPS = 1e-6  # M:37
PROB_CLAMP = 1e-7  # M:38
MODEL_MAGIC = b"FWM1"  # M:39
MODEL_VERSION = 1  # M:40
DEFAULT_MAX_SLOTS = 1 << 31  # M:41

_TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "u16": torch.uint16}
_WCODE = {"f32": _lib.W_F32, "bf16": _lib.W_BF16, "u16": _lib.W_U16Q}


@dataclass(frozen=True)
class ModelConfig:
    """Architecture + optimiser hyperparameters (M:44-110, same validation)."""

    n_fields: int
    k: int = 4
    hidden_sizes: tuple = ()
    lr_ffm: float = 0.05
    lr_lr: float = 0.05
    lr_nn: float = 0.01
    power_t: float = 0.5
    hash_bits: int = 18
    init_seed: int = 0
    init_scale_ffm: float = 0.5

    def __post_init__(self):
        object.__setattr__(self, "hidden_sizes", tuple(int(h) for h in self.hidden_sizes))
        if self.n_fields < 1:
            raise ContractError("n_fields must be >= 1")
        if self.k < 1:
            raise ContractError("k must be >= 1")
        if len(self.hidden_sizes) > 4:
            raise ContractError("at most 4 hidden layers are supported")
        if any(h < 1 for h in self.hidden_sizes):
            raise ContractError("hidden layer sizes must be positive")
        if min(self.lr_ffm, self.lr_lr, self.lr_nn) <= 0:
            raise ContractError("learning rates must be positive")
        if not 0.0 <= self.power_t <= 1.0:
            raise ContractError("power_t must lie in [0, 1]")
        if not 1 <= self.hash_bits <= 29:
            raise ContractError("hash_bits must lie in [1, 29]")
        if self.init_scale_ffm < 0:
            raise ContractError("init_scale_ffm must be >= 0")
        if not 0 <= self.init_seed < 1 << 64:
            raise ContractError("init_seed must fit in 64 bits")

    def to_json(self) -> str:
        d = {
            "n_fields": self.n_fields, "k": self.k, "hidden_sizes": list(self.hidden_sizes),
            "lr_ffm": self.lr_ffm, "lr_lr": self.lr_lr, "lr_nn": self.lr_nn,
            "power_t": self.power_t, "hash_bits": self.hash_bits, "init_seed": self.init_seed,
            "init_scale_ffm": self.init_scale_ffm,
        }
        return json.dumps(d, sort_keys=True, separators=(",", ":"))  # M:88-101

    @classmethod
    def from_json(cls, text: str) -> "ModelConfig":
        try:
            d = json.loads(text)
            d["hidden_sizes"] = tuple(d["hidden_sizes"])
            return cls(**d)
        except (ValueError, TypeError, KeyError) as exc:
            raise FormatError(f"bad model config payload: {exc}") from None


def pair_indices(n_fields: int):
    """Strict upper-triangle field pairs, row-major (M:113-117)."""
    iu, ju = np.triu_indices(n_fields, k=1)
    return iu.astype(np.int64), ju.astype(np.int64)


def pair_position(n_fields: int) -> np.ndarray:
    """(F, F) lookup from an unordered field pair to its output slot (M:120-127)."""
    iu, ju = pair_indices(n_fields)
    pos = np.full((n_fields, n_fields), -1, dtype=np.int64)
    pos[iu, ju] = np.arange(len(iu))
    pos[ju, iu] = pos[iu, ju]
    return pos


class WeightStore:
    """HBM-resident weight store (replaces M:142-230).

    ``wdtype`` selects the storage of the two hashed tables (``"f32"``,
    ``"bf16"`` -- the cfg5 large-table form -- or ``"u16"``, the paper's
    16-bit quantised form with per-table (min, bucket) headers).  The MLP is
    always f32.  ``version`` counts mutations exactly like M:155-158.
    """

    def __init__(self, config: ModelConfig, device=None, wdtype: str = "f32",
                 with_optimizer: bool = True, _alloc: bool = True):
        if wdtype not in _TORCH_DT:
            raise ContractError(f"unknown table dtype {wdtype!r}")
        self.config = config
        self.device = torch.device(device if device is not None else "cuda")
        self.wdtype = wdtype
        f, k = config.n_fields, config.k
        self.n_features = 1 << config.hash_bits
        self.n_pairs = f * (f - 1) // 2
        self.merged_width = 1 + self.n_pairs
        self.lr_size = self.n_features + 1
        self.ffm_size = self.n_features * f * k
        if config.hidden_sizes:
            dims = [self.merged_width, *config.hidden_sizes, 1]
            self.nn_dims = list(zip(dims[:-1], dims[1:]))
        else:
            self.nn_dims = []
        self.nn_size = sum(i * o + o for i, o in self.nn_dims)
        self.weights_total = self.lr_size + self.ffm_size + self.nn_size
        self.total_slots = 2 * self.weights_total
        # offsets of the blocks in the reference's flat layout (M:182-184)
        self.ffm_offset = self.lr_size
        self.nn_offset = self.ffm_offset + self.ffm_size
        self.acc_offset = self.weights_total
        self.pair_iu, self.pair_ju = pair_indices(f)
        self.version = 0
        self.q_headers = {}  # table name -> (w_min f32, bucket f32) for u16 stores
        self._cmodel = None
        self.lr = self.ffm = None
        self.nn_layers: list = []
        self.lr_acc = self.ffm_acc = None
        self.nn_accs: list = []
        if _alloc:
            dt = _TORCH_DT[wdtype]
            self.lr = torch.zeros(self.lr_size, dtype=dt, device=self.device)
            self.ffm = torch.zeros((self.n_features, f, k), dtype=dt, device=self.device)
            self.nn_layers = [(torch.zeros((i, o), dtype=torch.float32, device=self.device),
                               torch.zeros(o, dtype=torch.float32, device=self.device))
                              for i, o in self.nn_dims]
            if with_optimizer:
                if wdtype != "f32":
                    raise ContractError("only f32 stores carry optimizer state")
                # a bare store is all zeros, accumulators included (M:178-180);
                # init_model sets them to 1.0 (M:271)
                self.lr_acc = torch.zeros(self.lr_size, dtype=torch.float32, device=self.device)
                self.ffm_acc = torch.zeros((self.n_features, f, k), dtype=torch.float32,
                                           device=self.device)
                self.nn_accs = [(torch.zeros_like(w), torch.zeros_like(b))
                                for w, b in self.nn_layers]

    # ---------------------------------------------------------------- C view
    @property
    def has_optimizer(self) -> bool:
        return self.lr_acc is not None

    @property
    def bias(self) -> float:
        return float(self.lr[self.n_features].float().item())

    def c_model(self) -> _lib.DffmModel:
        """POD the C ABI consumes (include/dffm.h: dffm_model)."""
        m = _lib.DffmModel()
        m.n_fields = self.config.n_fields
        m.k = self.config.k
        m.hash_bits = self.config.hash_bits
        m.n_layers = len(self.nn_dims)
        dims = [self.merged_width, *self.config.hidden_sizes, 1] if self.nn_dims else []
        for i, d in enumerate(dims):
            m.dims[i] = d
        m.wdtype = _WCODE[self.wdtype]
        m.lr = self.lr.data_ptr()
        m.ffm = self.ffm.data_ptr()
        for i, (w, b) in enumerate(self.nn_layers):
            m.W[i] = w.data_ptr()
            m.b[i] = b.data_ptr()
        if self.wdtype == "u16":
            m.q_lr_min, m.q_lr_bucket = self.q_headers["lr"]
            m.q_ffm_min, m.q_ffm_bucket = self.q_headers["ffm"]
        return m

    def c_model_ref(self):
        self._cmodel = self.c_model()
        return ctypes.byref(self._cmodel)

    # ---------------------------------------------------------------- flat layout
    def blocks(self, include_optimizer=True):
        """(name, tensor) in the frozen flat order (M:145-153)."""
        out = [("lr", self.lr), ("ffm", self.ffm)]
        for i, (w, b) in enumerate(self.nn_layers):
            out += [(f"W{i}", w), (f"b{i}", b)]
        if include_optimizer:
            if not self.has_optimizer:
                raise ContractError("store has no optimizer state")
            out += [("lr_acc", self.lr_acc), ("ffm_acc", self.ffm_acc)]
            for i, (w, b) in enumerate(self.nn_accs):
                out += [(f"W{i}_acc", w), (f"b{i}_acc", b)]
        return out

    def weight_values(self, include_optimizer: bool = True) -> np.ndarray:
        """Host f32 copy of the flat array in layout order (M:218-221)."""
        parts = []
        for name, t in self.blocks(include_optimizer):
            parts.append(_to_f32_host(self, name, t).reshape(-1))
        return np.concatenate(parts)

    def load_flat(self, flat: np.ndarray) -> "WeightStore":
        """Fill the device blocks from a reference-layout flat f32 array."""
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        n_w = self.weights_total
        if flat.size not in (n_w, 2 * n_w):
            raise FormatError(f"flat payload holds {flat.size} values, layout wants "
                              f"{n_w} or {2 * n_w}")
        off = 0
        for name, t in self.blocks(include_optimizer=flat.size == 2 * n_w and self.has_optimizer):
            src = torch.from_numpy(flat[off:off + t.numel()]).view(t.shape)
            _from_f32(self, name, t, src)
            off += t.numel()
        if flat.size == n_w and self.has_optimizer:
            for _, t in self.blocks(True)[len(self.blocks(False)):]:
                t.fill_(1.0)  # M:682-683
        self.version += 1
        return self

    @classmethod
    def from_flat(cls, config, flat, device=None, wdtype="f32", with_optimizer=True):
        st = cls(config, device, wdtype, with_optimizer).load_flat(flat)
        st.version = 0  # a freshly built store, like WeightStore(config) (M:180)
        return st

    def copy(self) -> "WeightStore":
        dup = WeightStore(self.config, self.device, self.wdtype, _alloc=False)
        dup.lr, dup.ffm = self.lr.clone(), self.ffm.clone()
        dup.nn_layers = [(w.clone(), b.clone()) for w, b in self.nn_layers]
        if self.has_optimizer:
            dup.lr_acc, dup.ffm_acc = self.lr_acc.clone(), self.ffm_acc.clone()
            dup.nn_accs = [(w.clone(), b.clone()) for w, b in self.nn_accs]
        dup.q_headers = dict(self.q_headers)
        dup.version = self.version
        return dup

    def mark_mutated(self):
        self.version += 1

    def fill_accumulators(self, value: float = 1.0) -> "WeightStore":
        """Set every Adagrad accumulator to ``value`` (init_model uses 1.0, M:271)."""
        if not self.has_optimizer:
            raise ContractError("store has no optimizer state")
        for _, t in self.blocks(True)[len(self.blocks(False)):]:
            t.fill_(value)
        return self

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for _, t in self.blocks(self.has_optimizer))


def _to_f32_host(store: WeightStore, name: str, t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.float32:
        return t.detach().cpu().numpy()
    if t.dtype == torch.bfloat16:
        return t.detach().float().cpu().numpy()
    from .quant import dequantize_tensor  # u16 table -> f32 (bit-exact K4)
    hmin, hb = store.q_headers[name]
    return dequantize_tensor(t, hmin, hb).cpu().numpy()


def _from_f32(store: WeightStore, name: str, dst: torch.Tensor, src: torch.Tensor):
    if dst.dtype == torch.uint16:
        raise ContractError("load a u16 store through quant.quantize_store")
    dst.copy_(src.to(dst.dtype) if dst.dtype != torch.float32 else src, non_blocking=False)


# --------------------------------------------------------------------------- init


def init_model(config: ModelConfig, max_slots: int = DEFAULT_MAX_SLOTS, device=None,
               chunk: int = 1 << 24) -> WeightStore:
    """Deterministic init, bit-identical to M:233-272.

    The reference draws ``rng.random(ffm_size)`` then ``rng.uniform`` per MLP
    layer from one ``default_rng(init_seed)``; drawing the same streams in
    chunks reproduces them bit for bit without the multi-GB f64 temporary."""
    f, k = config.n_fields, config.k
    n_features = 1 << config.hash_bits
    merged = 1 + f * (f - 1) // 2
    nn = 0
    if config.hidden_sizes:
        dims = [merged, *config.hidden_sizes, 1]
        nn = sum(i * o + o for i, o in zip(dims[:-1], dims[1:]))
    total = 2 * (n_features + 1 + n_features * f * k + nn)
    if total > max_slots:
        raise SizingError(f"model wants {total} float32 slots, cap is {max_slots};"
                          " lower hash_bits, k, or the layer widths")  # M:248-253
    store = WeightStore(config, device)
    store.fill_accumulators(1.0)  # M:271
    rng = np.random.default_rng(config.init_seed)
    if config.init_scale_ffm > 0:
        scale = config.init_scale_ffm / math.sqrt(k)
        flat_ffm = store.ffm.view(-1)
        for c0 in range(0, store.ffm_size, chunk):
            c1 = min(store.ffm_size, c0 + chunk)
            vals = (scale * (1.0 - rng.random(c1 - c0))).astype(np.float32)
            flat_ffm[c0:c1].copy_(torch.from_numpy(vals))
    for (i_dim, o_dim), (w, _) in zip(store.nn_dims, store.nn_layers):
        limit = math.sqrt(6.0 / (i_dim + o_dim))
        vals = rng.uniform(-limit, limit, i_dim * o_dim).astype(np.float32)
        w.view(-1).copy_(torch.from_numpy(vals))
    return store


# --------------------------------------------------------------------------- forward


class OpCounter:
    """Counts multiply-add units in interaction-block inner loops (M:130-139)."""

    __slots__ = ("madds",)

    def __init__(self):
        self.madds = 0

    def add(self, n: int):
        self.madds += int(n)


@dataclass
class ForwardState:
    """Per-example intermediates kept for the backward pass (M:275-290).

    ``forward`` fills every field from the K11 device trace (f64); the batched
    paths (K1 / K2) keep these on chip and never materialise them."""

    lr_out: float
    ffm_pair_outputs: np.ndarray  # float64 (n_pairs,)
    merged_input: np.ndarray  # float64 (1 + n_pairs,)
    layer_pre_acts: list
    layer_acts: list
    logit: float
    latent_sums: np.ndarray = field(repr=False, default=None)  # (F, F, k)
    merge_vec: np.ndarray = field(repr=False, default=None)
    merge_mu: float = 0.0
    merge_sd: float = 0.0
    _store: "WeightStore" = field(repr=False, default=None)
    _store_version: int = 0


def _sigmoid(logit: float) -> float:
    if logit >= 0:
        return 1.0 / (1.0 + math.exp(-min(logit, 60.0)))
    e = math.exp(max(logit, -60.0))
    return e / (1.0 + e)


def predict_proba(logit: float) -> float:
    """Sigmoid clamped to [1e-7, 1 - 1e-7] (M:300-305)."""
    if not math.isfinite(logit):
        raise NumericError("non-finite logit", block="logit")
    p = _sigmoid(logit)
    return min(max(p, PROB_CLAMP), 1.0 - PROB_CLAMP)


def _as_device(x, dtype, device):
    if isinstance(x, torch.Tensor):
        t = x if x.device == device else x.to(device, non_blocking=True)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(device)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


class StatusWord:
    """Device status word (include/dffm.h) with a pinned host mirror."""

    def __init__(self, device):
        # int64 storage holding the uint64 bit pattern; all-ones = clear
        self.dev = torch.empty(1, dtype=torch.int64, device=device)
        self.host = torch.empty(1, dtype=torch.int64, pin_memory=True)

    def clear(self):
        self.dev.fill_(-1)

    def ptr(self):
        return self.dev.data_ptr()

    def fetch_async(self):
        self.host.copy_(self.dev, non_blocking=True)

    def raise_if_set(self, what="", base=0):
        _lib.raise_status(int(self.host.item()) & ((1 << 64) - 1), what, base)


_status_cache: dict = {}


def _status(device) -> StatusWord:
    key = (device.type, device.index)
    if key not in _status_cache:
        _status_cache[key] = StatusWord(device)
    return _status_cache[key]


def predict_batch(idx, val, store: WeightStore, out: torch.Tensor | None = None,
                  logits: torch.Tensor | None = None, check: bool = True,
                  stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """K1 over a padded batch: idx int32 [n,F,M] (-1 empty), val f32 [n,F,M].

    Returns device f32 probabilities [n] (M:300-305 applied); with ``check``
    the device status word is read back and the first non-finite example
    raises ``NumericError(block=...)`` exactly as M:392-396 would."""
    dev = store.device
    idx = _as_device(idx, torch.int32, dev)
    val = _as_device(val, torch.float32, dev)
    if idx.dim() != 3 or idx.shape != val.shape or idx.shape[1] != store.config.n_fields:
        raise ContractError(f"expected idx/val [n, {store.config.n_fields}, M], got "
                            f"{tuple(idx.shape)} / {tuple(val.shape)}")
    n, _, M = idx.shape
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    st = _status(dev)
    cur = torch.cuda.current_stream(dev)
    s = stream if stream is not None else cur
    if s != cur:
        s.wait_stream(cur)  # inputs/outputs were staged on the current stream
    with torch.cuda.stream(s):
        st.clear()
        rc = _lib.lib().dffm_forward(store.c_model_ref(), idx.data_ptr(), val.data_ptr(), M, n,
                                     out.data_ptr(), logits.data_ptr() if logits is not None
                                     else None, 0, st.ptr(), s.cuda_stream)
        _lib.check(rc, "dffm_forward")
        if check:
            st.fetch_async()
    if check:
        s.synchronize()
        st.raise_if_set("forward: ")
    return out


def _chunk_bounds(n: int, chunk: int):
    """[c0, c1) chunks of a host batch: sizes ramp up chunk/8, chunk/4, ...,
    chunk so the first (unoverlapped) host->device copy is short."""
    out, c0, sz = [], 0, max(1, chunk // 8)
    while c0 < n:
        c1 = min(n, c0 + sz)
        out.append((c0, c1))
        c0, sz = c1, min(chunk, sz * 2)
    return out


class HostPredictor:
    """Public host-buffer entry point: pinned host idx/val in, host probs out.

    The batch is cut into chunks; chunk i+1's H2D copy (copy stream) overlaps
    chunk i's K1 launch and its 4 B/example D2H (compute stream), with two
    device staging buffers in flight.  This is the path a serving caller
    with host-resident requests uses (and the bench's ``e2e`` number)."""

    def __init__(self, store: WeightStore, max_examples: int, max_per_field: int,
                 chunk: int = 1 << 17):
        self.store = store
        self.chunk = int(min(chunk, max(1, max_examples)))
        F = store.config.n_fields
        dev = store.device
        self.idx_buf = [torch.empty((self.chunk, F, max_per_field), dtype=torch.int32, device=dev)
                        for _ in range(2)]
        self.val_buf = [torch.empty((self.chunk, F, max_per_field), dtype=torch.float32,
                                    device=dev) for _ in range(2)]
        self.prob_buf = [torch.empty(self.chunk, dtype=torch.float32, device=dev)
                         for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(dev)
        self.compute_stream = torch.cuda.Stream(dev)
        self.status = StatusWord(dev)
        self.launches = 0

    def __call__(self, idx_host: torch.Tensor, val_host: torch.Tensor,
                 out_host: torch.Tensor, check: bool = True) -> torch.Tensor:
        n, F, M = idx_host.shape
        lib = _lib.lib()
        cm = self.store.c_model_ref()
        cs, ks = self.copy_stream, self.compute_stream
        # order K1 after whatever the caller queued on its current stream
        # (weight writes, quantize_store, in-place edits of the tables)
        ks.wait_stream(torch.cuda.current_stream(self.store.device))
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        with torch.cuda.stream(ks):
            self.status.clear()
        cs.wait_stream(ks)
        for i, (c0, c1) in enumerate(_chunk_bounds(n, self.chunk)):
            b = i & 1
            ib = self.idx_buf[b][: c1 - c0]
            vb = self.val_buf[b][: c1 - c0]
            pb = self.prob_buf[b][: c1 - c0]
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(free[b])
                ib.copy_(idx_host[c0:c1], non_blocking=True)
                vb.copy_(val_host[c0:c1], non_blocking=True)
                h2d_done[b].record(cs)
            with torch.cuda.stream(ks):
                ks.wait_event(h2d_done[b])
                rc = lib.dffm_forward(cm, ib.data_ptr(), vb.data_ptr(), M, c1 - c0,
                                      pb.data_ptr(), None, c0, self.status.ptr(), ks.cuda_stream)
                _lib.check(rc, "dffm_forward")
                self.launches += 1
                out_host[c0:c1].copy_(pb, non_blocking=True)
                free[b].record(ks)
        with torch.cuda.stream(ks):
            self.status.fetch_async()
        ks.synchronize()
        if check:
            self.status.raise_if_set("forward: ")
        return out_host


    def predict_ragged(self, batch, out_host: torch.Tensor, check: bool = True) -> torch.Tensor:
        """Host-buffer entry point for ragged batches (``features.RaggedBatch``
        of pinned torch tensors): per chunk the present features only are
        copied (ex_off, cnt, idx, val slices), K9 (``dffm_unpack_ragged``)
        expands them to the padded layout in HBM and K1 scores them; copies of
        chunk i+1 overlap chunk i's kernels, as in ``__call__``."""
        n, F = int(batch.cnt.shape[0]), int(batch.cnt.shape[1])
        M = batch.max_per_field
        lib = _lib.lib()
        cm = self.store.c_model_ref()
        cs, ks = self.copy_stream, self.compute_stream
        # order K1 after whatever the caller queued on its current stream
        # (weight writes, quantize_store, in-place edits of the tables)
        ks.wait_stream(torch.cuda.current_stream(self.store.device))
        dev = self.store.device
        if not hasattr(self, "rg_off"):
            self.rg_off = [torch.empty(self.chunk + 1, dtype=torch.int64, device=dev)
                           for _ in range(2)]
            self.rg_cnt = [torch.empty((self.chunk, F), dtype=torch.uint8, device=dev)
                           for _ in range(2)]
            self.rg_cap = 0
        off_h = batch.ex_off
        bounds = _chunk_bounds(n, self.chunk)
        nnz_max = max(int(off_h[c1]) - int(off_h[c0]) for c0, c1 in bounds) if bounds else 0
        if nnz_max > self.rg_cap:
            self.rg_cap = nnz_max
            self.rg_idx = [torch.empty(nnz_max, dtype=torch.int32, device=dev) for _ in range(2)]
            self.rg_val = [torch.empty(nnz_max, dtype=torch.float32, device=dev) for _ in range(2)]
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        with torch.cuda.stream(ks):
            self.status.clear()
        cs.wait_stream(ks)
        for i, (c0, c1) in enumerate(bounds):
            b = i & 1
            z0, z1 = int(off_h[c0]), int(off_h[c1])
            ob, cb = self.rg_off[b][: c1 - c0 + 1], self.rg_cnt[b][: c1 - c0]
            ib, vb = self.rg_idx[b][: z1 - z0], self.rg_val[b][: z1 - z0]
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(free[b])
                ob.copy_(off_h[c0:c1 + 1], non_blocking=True)
                cb.copy_(batch.cnt[c0:c1], non_blocking=True)
                ib.copy_(batch.idx[z0:z1], non_blocking=True)
                vb.copy_(batch.val[z0:z1], non_blocking=True)
                h2d_done[b].record(cs)
            pi = self.idx_buf[b][: c1 - c0]
            pv = self.val_buf[b][: c1 - c0]
            pb = self.prob_buf[b][: c1 - c0]
            with torch.cuda.stream(ks):
                ks.wait_event(h2d_done[b])
                _lib.check(lib.dffm_unpack_ragged(ob.data_ptr(), cb.data_ptr(), ib.data_ptr(),
                                                  vb.data_ptr(), c1 - c0, F, M, z0,
                                                  pi.data_ptr(), pv.data_ptr(), c0,
                                                  self.status.ptr(), ks.cuda_stream),
                           "dffm_unpack_ragged")
                rc = lib.dffm_forward(cm, pi.data_ptr(), pv.data_ptr(), M, c1 - c0,
                                      pb.data_ptr(), None, c0, self.status.ptr(), ks.cuda_stream)
                _lib.check(rc, "dffm_forward")
                self.launches += 1
                out_host[c0:c1].copy_(pb, non_blocking=True)
                free[b].record(ks)
        with torch.cuda.stream(ks):
            self.status.fetch_async()
        ks.synchronize()
        if check:
            self.status.raise_if_set("forward: ")
        return out_host


    def predict_packed(self, batch, out_host: torch.Tensor, check: bool = True) -> torch.Tensor:
        """Host-buffer entry point for ``features.PackedBatch`` (pinned torch
        tensors): per chunk the packed slices are copied, K9b
        (``dffm_unpack_packed``) expands them to the padded layout, K1 scores."""
        n, F = int(batch.cnt.shape[0]), int(batch.cnt.shape[1])
        M = batch.max_per_field
        W = batch.idx_width
        lib = _lib.lib()
        cm = self.store.c_model_ref()
        cs, ks = self.copy_stream, self.compute_stream
        # order K1 after whatever the caller queued on its current stream
        # (weight writes, quantize_store, in-place edits of the tables)
        ks.wait_stream(torch.cuda.current_stream(self.store.device))
        dev = self.store.device
        bounds = _chunk_bounds(n, self.chunk)
        off_h, voff_h = batch.ex_off, batch.voff
        zs = [(int(off_h[c0]), int(off_h[c1]), int(voff_h[c0]), int(voff_h[c1])) for c0, c1 in bounds]
        need = (max((z1 - z0 for z0, z1, _, _ in zs), default=0),
                max((v1 - v0 for _, _, v0, v1 in zs), default=0))
        if getattr(self, "pk_cap", None) != need:
            self.pk_off = [torch.empty(self.chunk + 1, dtype=torch.int64, device=dev) for _ in range(2)]
            self.pk_voff = [torch.empty(self.chunk + 1, dtype=torch.int64, device=dev) for _ in range(2)]
            self.pk_cnt = [torch.empty((self.chunk, F), dtype=torch.uint8, device=dev) for _ in range(2)]
            self.pk_idx = [torch.empty(need[0] * 4 + 8, dtype=torch.uint8, device=dev) for _ in range(2)]
            self.pk_bits = [torch.empty(need[0] // 8 + 16, dtype=torch.uint8, device=dev) for _ in range(2)]
            self.pk_vals = [torch.empty(need[1] + 1, dtype=torch.float32, device=dev) for _ in range(2)]
            self.pk_cap = need
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        with torch.cuda.stream(ks):
            self.status.clear()
        cs.wait_stream(ks)
        for i, ((c0, c1), (z0, z1, v0, v1)) in enumerate(zip(bounds, zs)):
            b = i & 1
            y0, y1 = z0 // 8, (z1 + 7) // 8
            ob, vob = self.pk_off[b][: c1 - c0 + 1], self.pk_voff[b][: c1 - c0 + 1]
            cb = self.pk_cnt[b][: c1 - c0]
            ib = self.pk_idx[b][: (z1 - z0) * W]
            bb = self.pk_bits[b][: y1 - y0]
            vb = self.pk_vals[b][: v1 - v0]
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(free[b])
                ob.copy_(off_h[c0:c1 + 1], non_blocking=True)
                vob.copy_(voff_h[c0:c1 + 1], non_blocking=True)
                cb.copy_(batch.cnt[c0:c1], non_blocking=True)
                ib.copy_(batch.idx_bytes[z0 * W:z1 * W], non_blocking=True)
                bb.copy_(batch.vbits[y0:y1], non_blocking=True)
                vb.copy_(batch.vals[v0:v1], non_blocking=True)
                h2d_done[b].record(cs)
            pi = self.idx_buf[b][: c1 - c0]
            pv = self.val_buf[b][: c1 - c0]
            pb = self.prob_buf[b][: c1 - c0]
            with torch.cuda.stream(ks):
                ks.wait_event(h2d_done[b])
                _lib.check(lib.dffm_unpack_packed(ob.data_ptr(), cb.data_ptr(), ib.data_ptr(), W,
                                                  bb.data_ptr(), vb.data_ptr(), vob.data_ptr(),
                                                  c1 - c0, F, M, z0, z0 - 8 * y0, v0,
                                                  pi.data_ptr(), pv.data_ptr(), c0,
                                                  self.status.ptr(), ks.cuda_stream),
                           "dffm_unpack_packed")
                rc = lib.dffm_forward(cm, pi.data_ptr(), pv.data_ptr(), M, c1 - c0,
                                      pb.data_ptr(), None, c0, self.status.ptr(), ks.cuda_stream)
                _lib.check(rc, "dffm_forward")
                self.launches += 1
                out_host[c0:c1].copy_(pb, non_blocking=True)
                free[b].record(ks)
        with torch.cuda.stream(ks):
            self.status.fetch_async()
        ks.synchronize()
        if check:
            self.status.raise_if_set("forward: ")
        return out_host


def _example_arrays(example, store: WeightStore):
    """One ParsedExample-like object -> padded device idx/val [1, F, M] (M >= 1);
    a field id >= F is the ContractError of M:331-334."""
    f_count = store.config.n_fields
    m = 1
    for ff in example.fields:
        if ff.field_id >= f_count:
            raise ContractError(f"field id {ff.field_id} outside model's {f_count} fields")
        m = max(m, len(ff.indices))
    idx = np.full((1, f_count, m), -1, np.int32)
    val = np.zeros((1, f_count, m), np.float32)
    for ff in example.fields:
        n = len(ff.indices)
        if n:
            idx[0, ff.field_id, :n] = np.asarray(ff.indices, np.int64)
            val[0, ff.field_id, :n] = np.asarray(ff.values, np.float64)
    return (torch.from_numpy(idx).to(store.device), torch.from_numpy(val).to(store.device))


def _count_macs(example, store: WeightStore, state: ForwardState, counter: OpCounter):
    """M:340-341, M:352-353, M:374-375: the reference's MAC accounting."""
    f_count, k = store.config.n_fields, store.config.k
    present = set()
    for ff in example.fields:
        m = len(ff.indices)
        if m:
            counter.add(m + m * f_count * k)
            present.add(ff.field_id)
    n_active = sum(1 for a, b in zip(store.pair_iu, store.pair_ju)
                   if a in present and b in present)
    if n_active:
        counter.add(n_active * k)
    if store.nn_dims:
        counter.add(sum(i * o for i, o in store.nn_dims))


def _diagnose_nonfinite(state: ForwardState) -> str:
    """First non-finite stage in the order lr, ffm, merge, nn, logit (M:308-318)."""
    if not math.isfinite(state.lr_out):
        return "lr"
    if not np.isfinite(state.ffm_pair_outputs).all():
        return "ffm"
    if not np.isfinite(state.merged_input).all():
        return "merge"
    for z in state.layer_pre_acts:
        if not np.isfinite(z).all():
            return "nn"
    return "logit"


def _trace(store: WeightStore, idx: torch.Tensor, val: torch.Tensor) -> torch.Tensor:
    lib = _lib.lib()
    cm = store.c_model_ref()
    n = int(lib.dffm_trace_len(cm))
    if n < 0:
        _lib.check(_lib.CONTRACT, "dffm_trace_len")
    out = torch.empty(n, dtype=torch.float64, device=store.device)
    s = torch.cuda.current_stream(store.device)
    _lib.check(lib.dffm_forward_trace(cm, idx.data_ptr(), val.data_ptr(), idx.shape[2],
                                      out.data_ptr(), s.cuda_stream), "dffm_forward_trace")
    return out


def forward(example, store: WeightStore, mac_counter: OpCounter | None = None) -> ForwardState:
    """One example through every block, keeping the intermediates (M:321-397).

    K11 (csrc/trace.cu) computes the reference's stages in f64 on the device:
    LR sum, latent sums S (F, F, k), DiagMask pairs, MergeNorm, the MLP layer
    by layer, the residual logit.  Read-only on the store; a non-finite logit
    raises NumericError(block=...) with the reference's diagnosis order."""
    idx, val = _example_arrays(example, store)
    tr = _trace(store, idx, val).cpu().numpy()
    cfg = store.config
    f_count, k, P, D = cfg.n_fields, cfg.k, store.n_pairs, store.merged_width
    o = _lib.TRACE_HEAD
    S = tr[o:o + f_count * f_count * k].reshape(f_count, f_count, k)
    o += f_count * f_count * k
    pairs = tr[o:o + P]
    v = tr[o + P:o + P + D]
    merged = tr[o + P + D:o + P + 2 * D]
    o += P + 2 * D
    pre, acts = [], []
    for _, width in store.nn_dims[:-1]:
        pre.append(tr[o:o + width].copy())
        acts.append(tr[o + width:o + 2 * width].copy())
        o += 2 * width
    state = ForwardState(lr_out=float(tr[0]), ffm_pair_outputs=pairs.copy(),
                         merged_input=merged.copy(), layer_pre_acts=pre, layer_acts=acts,
                         logit=float(tr[1]), latent_sums=S.copy(), merge_vec=v.copy(),
                         merge_mu=float(tr[2]), merge_sd=float(tr[3]), _store=store,
                         _store_version=store.version)
    if mac_counter is not None:
        _count_macs(example, store, state, mac_counter)
    if not math.isfinite(state.logit):
        blk = _diagnose_nonfinite(state)
        raise NumericError(f"non-finite value in {blk} block", block=blk)
    return state


def backward_update(state: ForwardState, example, label: int, store: WeightStore,
                    sparse: bool = True) -> float:
    """Backpropagate one example and apply the Adagrad updates in place
    (M:440-533); returns the example's log-loss and bumps ``store.version``.

    The step runs in K2 (csrc/train.cu), the same kernel as the batched trainer:
    it recomputes the forward pass on chip (identical to ``state``), merges
    duplicate buckets in occurrence order and applies the f64 Adagrad rule."""
    if state._store is not store or state._store_version != store.version:
        raise ContractError("forward state was not produced against this store state")
    if label not in (0, 1):
        raise ContractError(f"label must be 0 or 1, got {label!r}")
    from .training import _train_one
    p = _train_one(example, label, store, sparse)
    return -math.log(p) if label else -math.log1p(-p)


def loss_gradients(state: ForwardState, example, label: int, store: WeightStore) -> np.ndarray:
    """Dense float64 gradient of the log-loss over the weights' flat layout
    (M:575-634; lr | ffm | per layer W, b -- no accumulator block), computed
    by K11 on the device from the example's trace."""
    if state._store is not store or state._store_version != store.version:
        raise ContractError("forward state was not produced against this store state")
    if label not in (0, 1):
        raise ContractError(f"label must be 0 or 1, got {label!r}")
    idx, val = _example_arrays(example, store)
    tr = _trace(store, idx, val)
    lib = _lib.lib()
    cm = store.c_model_ref()
    grad = torch.empty(store.weights_total, dtype=torch.float64, device=store.device)
    scratch = torch.empty(max(1, int(lib.dffm_grad_scratch_len(cm))), dtype=torch.float64,
                          device=store.device)
    s = torch.cuda.current_stream(store.device)
    _lib.check(lib.dffm_loss_gradients(cm, idx.data_ptr(), val.data_ptr(), idx.shape[2],
                                       tr.data_ptr(), int(label), grad.data_ptr(),
                                       store.weights_total, scratch.data_ptr(), s.cuda_stream),
               "dffm_loss_gradients")
    return grad.cpu().numpy()


# --------------------------------------------------------------------------- serialisation


def _header_bytes(config: ModelConfig, include_optimizer: bool) -> bytes:
    payload = config.to_json().encode("utf-8")
    return (MODEL_MAGIC + MODEL_VERSION.to_bytes(4, "little") + len(payload).to_bytes(4, "little")
            + payload + bytes([1 if include_optimizer else 0]))  # M:640-648


def flat_weight_view(store: WeightStore, include_optimizer: bool = True) -> bytes:
    """Header + flat little-endian f32 block, byte-identical to M:651-660."""
    values = store.weight_values(include_optimizer)
    return _header_bytes(store.config, include_optimizer) + values.astype("<f4", copy=False).tobytes()


def store_from_bytes(data: bytes, device=None) -> WeightStore:
    """Parse M:663-684's format into a device store."""
    if data[:4] != MODEL_MAGIC:
        raise FormatError("not a model file (bad magic)")
    version = int.from_bytes(data[4:8], "little")
    if version != MODEL_VERSION:
        raise FormatError(f"unsupported model file version {version}")
    n = int.from_bytes(data[8:12], "little")
    if len(data) < 12 + n + 1:
        raise FormatError("truncated model header")
    config = ModelConfig.from_json(data[12:12 + n].decode("utf-8"))
    has_opt = data[12 + n] == 1
    body = np.frombuffer(data[13 + n:], dtype="<f4")
    store = WeightStore(config, device)
    expected = store.total_slots if has_opt else store.weights_total
    if len(body) != expected:
        raise FormatError(f"weight payload holds {len(body)} values, layout wants {expected}")
    store.load_flat(body.astype(np.float32))
    store.version = 0
    return store


def save_model(store: WeightStore, path, include_optimizer: bool = True):
    with open(path, "wb") as fh:
        fh.write(flat_weight_view(store, include_optimizer))


def load_model(path, device=None) -> WeightStore:
    with open(path, "rb") as fh:
        return store_from_bytes(fh.read(), device)
