"""Canonical examples <-> the padded GPU batch layout.

The reference's canonical example (Fe:121-172) is a label plus, per present
field, strictly increasing int64 indices with f64 values (duplicates summed,
Fe:219).  The device layout is a dense padded batch:

    idx [n][F][M] int32   field f's indices in slots 0..m_f-1, then -1
    val [n][F][M] f32     matching values, 0 in empty slots
    labels [n] uint8

with fields at their field-id position, so "field order" on the device is
ascending field id (the f64 lr sum of M:338 is order-insensitive at the
1e-16 level).  Values are rounded to f32 on the way in; the synthetic
workloads only produce f32-representable values, so both sides see identical
inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ContractError


def transform_numeric(v: float) -> float:
    """ln(1+v) for v > 0, else v (Fe:33-39); K10 applies it on the device for
    the numeric fields of parsed text."""
    return math.log1p(v) if v > 0 else v


@dataclass(frozen=True)
class FieldFeatures:
    """Features of one field: sorted unique hashed indices (int64) and their
    f64 values (Fe:121-143)."""

    field_id: int
    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.indices.flags.writeable = False
        self.values.flags.writeable = False

    def __eq__(self, other):
        return (isinstance(other, FieldFeatures) and self.field_id == other.field_id
                and np.array_equal(self.indices, other.indices)
                and np.array_equal(self.values, other.values))

    def __len__(self) -> int:
        return len(self.indices)


@dataclass(frozen=True)
class ParsedExample:
    """One labeled instance: binary label plus per-field hashed features in the
    order the fields first appear (Fe:145-157)."""

    label: int
    fields: tuple

    def __eq__(self, other):
        return (isinstance(other, ParsedExample) and self.label == other.label
                and self.fields == other.fields)


def pack_examples(examples, n_fields: int, max_per_field: int | None = None):
    """ParsedExample-like objects (``.label``, ``.fields[i].field_id/.indices/
    .values``) -> (idx int32 [n,F,M], val f32 [n,F,M], labels uint8 [n])."""
    rows = []
    mmax = 1
    for ex in examples:
        per = {}
        for ff in ex.fields:
            fid = int(ff.field_id)
            if fid < 0 or fid >= n_fields:
                raise ContractError(f"field id {fid} outside model's {n_fields} fields")  # M:331
            ix = np.asarray(ff.indices, dtype=np.int64)
            vx = np.asarray(ff.values, dtype=np.float64)
            if fid in per:  # repeated field block: merge like Fe:185-219
                ix = np.concatenate([per[fid][0], ix])
                vx = np.concatenate([per[fid][1], vx])
            per[fid] = (ix, vx)
        canon = {}
        for fid, (ix, vx) in per.items():
            u, inv = np.unique(ix, return_inverse=True)
            v = np.zeros(len(u))
            np.add.at(v, inv, vx)
            canon[fid] = (u, v)
            mmax = max(mmax, len(u))
        rows.append((int(getattr(ex, "label", 0)), canon))
    M = mmax if max_per_field is None else max_per_field
    if mmax > M:
        raise ContractError(f"a field holds {mmax} features, max_per_field is {M}")
    n = len(rows)
    idx = np.full((n, n_fields, M), -1, np.int32)
    val = np.zeros((n, n_fields, M), np.float32)
    labels = np.zeros(n, np.uint8)
    for e, (lab, canon) in enumerate(rows):
        labels[e] = 1 if lab == 1 else 0
        if lab not in (0, 1):
            raise ContractError(f"label must be 0 or 1, got {lab!r}")  # M:453-454
        for fid, (u, v) in canon.items():
            if len(u) and (u.min() < 0 or u.max() >= np.iinfo(np.int32).max):
                raise ContractError("feature index out of range")
            idx[e, fid, :len(u)] = u
            val[e, fid, :len(u)] = v
    return idx, val, labels


def unpack_row(idx_row, val_row):
    """One padded row -> [(field_id, int64 indices, f64 values)] in field order."""
    out = []
    for f in range(idx_row.shape[0]):
        sel = idx_row[f] >= 0
        if sel.any():
            out.append((f, idx_row[f][sel].astype(np.int64), val_row[f][sel].astype(np.float64)))
    return out


class RaggedBatch:
    """The batched canonical form of ParsedExamples (Fe:121-172), CSR over
    (example, field): ``ex_off`` int64 [n+1] (example e's features are
    ``idx[ex_off[e]:ex_off[e+1]]``), ``cnt`` uint8 [n, F] (features per field,
    0 = absent), ``idx`` int32 / ``val`` float32 [nnz] in example, field, slot
    order.  It carries only present features, so it is the cheaper host->device
    format when fields are sparse (cfg2: 47.4 of 72 padded slots) --
    ``dffm_unpack_ragged`` (K9) expands it to the padded layout on the device.
    Arrays may be numpy or (pinned) torch tensors."""

    def __init__(self, ex_off, cnt, idx, val, max_per_field: int):
        self.ex_off, self.cnt, self.idx, self.val = ex_off, cnt, idx, val
        self.max_per_field = int(max_per_field)

    @property
    def n(self) -> int:
        return int(self.cnt.shape[0])

    @property
    def n_fields(self) -> int:
        return int(self.cnt.shape[1])

    def nbytes(self) -> int:
        return sum(int(a.nbytes if hasattr(a, "nbytes") else a.numel() * a.element_size())
                   for a in (self.ex_off, self.cnt, self.idx, self.val))

    @classmethod
    def from_padded(cls, idx, val) -> "RaggedBatch":
        """Padded [n, F, M] (slots 0..m_f-1 live, then -1) -> ragged (numpy)."""
        idx = np.asarray(idx)
        val = np.asarray(val)
        n, F, M = idx.shape
        live = idx >= 0
        cnt = live.sum(axis=2).astype(np.uint8)
        ex_off = np.zeros(n + 1, np.int64)
        np.cumsum(cnt.sum(axis=1, dtype=np.int64), out=ex_off[1:])
        return cls(ex_off, cnt, np.ascontiguousarray(idx[live], dtype=np.int32),
                   np.ascontiguousarray(val[live], dtype=np.float32), M)

    @classmethod
    def from_examples(cls, examples, n_fields: int, max_per_field: int | None = None):
        idx, val, labels = pack_examples(examples, n_fields, max_per_field)
        return cls.from_padded(idx, val), labels

    def to_padded(self):
        """Host-side inverse (tests): -> (idx int32 [n,F,M], val f32 [n,F,M])."""
        cnt = np.asarray(self.cnt)
        n, F = cnt.shape
        M = self.max_per_field
        idx = np.full((n, F, M), -1, np.int32)
        val = np.zeros((n, F, M), np.float32)
        live = np.arange(M)[None, None, :] < cnt[:, :, None]
        idx[live] = np.asarray(self.idx)
        val[live] = np.asarray(self.val)
        return idx, val


class PackedBatch:
    """Wire format for host-resident batches (K9b unpacks it on the device): the
    ragged batch with each bucket index in ``idx_width`` little-endian bytes (3
    when every index < 2^24 -- exact) and the values equal to 1.0 (categorical
    indicators, Fe:202) elided: bit t of ``vbits`` (LSB first) says feature t
    carries an explicit f32 in ``vals``; ``voff`` int64 [n+1] indexes ``vals``
    per example.  cfg2: ~215 B per example vs 411 B ragged, 576 B padded."""

    def __init__(self, ex_off, cnt, idx_bytes, idx_width, vbits, vals, voff, max_per_field):
        self.ex_off, self.cnt, self.idx_bytes, self.vbits = ex_off, cnt, idx_bytes, vbits
        self.vals, self.voff = vals, voff
        self.idx_width, self.max_per_field = int(idx_width), int(max_per_field)

    @property
    def n(self) -> int:
        return int(self.cnt.shape[0])

    def nbytes(self) -> int:
        return sum(int(a.nbytes if hasattr(a, "nbytes") else a.numel() * a.element_size())
                   for a in (self.ex_off, self.cnt, self.idx_bytes, self.vbits, self.vals,
                             self.voff))

    @classmethod
    def from_ragged(cls, rb: "RaggedBatch") -> "PackedBatch":
        idx = np.asarray(rb.idx, np.int64)
        val = np.asarray(rb.val, np.float32)
        width = 3 if (len(idx) == 0 or idx.max() < (1 << 24)) else 4
        if len(idx) and idx.min() < 0:
            raise ContractError("negative bucket index in a ragged batch")
        ib = idx.astype("<u4").view(np.uint8).reshape(-1, 4)[:, :width]
        explicit = ~(val.view(np.uint32) == np.float32(1.0).view(np.uint32))  # bit-exact 1.0
        vbits = np.packbits(explicit, bitorder="little")
        ex_off = np.asarray(rb.ex_off, np.int64)
        cs = np.concatenate([[0], np.cumsum(explicit, dtype=np.int64)])
        return cls(ex_off, np.asarray(rb.cnt, np.uint8), np.ascontiguousarray(ib).ravel(), width,
                   vbits, np.ascontiguousarray(val[explicit]), cs[ex_off], rb.max_per_field)


# --------------------------------------------------------------------------- text input (K10)

MIN_HASH_BITS, MAX_HASH_BITS = 10, 29  # H:24-25

PARSE_ERRORS = {
    1: "malformed label (want 0, 1, or -1)",        # Fe:229
    2: "example has no field blocks",               # Fe:231
    3: "empty field block (missing field name after '|')",  # Fe:191
    4: "unknown field name",                        # InputSchema.field_id
    5: "bad value",                                 # Fe:203-205
    6: "non-finite value",                          # Fe:206-207
    7: "raw index out of range for hash_bits",      # Fe:211-214
    8: "non-ASCII whitespace or digits (not supported by the GPU parser)",
    9: "more than 1024 features in one line (GPU parser limit)",
    10: "more than 255 features in one field (GPU parser limit)",
    11: "blank line",  # skipped by the reference's stream loops (T:176, T:227)
}


class InputSchema:
    """Ordered field list + numeric flags + hash_bits (API of the reference's
    InputSchema, Fe:42-118: same validation, from_text/to_text format)."""

    def __init__(self, field_names, numeric_fields=frozenset(), hash_bits: int = 18):
        from .errors import ParseError
        self.field_names = tuple(field_names)
        self.numeric_fields = frozenset(numeric_fields)
        self.hash_bits = int(hash_bits)
        if not self.field_names:
            raise ParseError("schema declares no fields")
        if len(set(self.field_names)) != len(self.field_names):
            raise ParseError("schema field names must be unique")
        if not MIN_HASH_BITS <= self.hash_bits <= MAX_HASH_BITS:
            raise ParseError(f"hash_bits must be in [{MIN_HASH_BITS}, {MAX_HASH_BITS}],"
                             f" got {self.hash_bits}")
        unknown = self.numeric_fields - set(self.field_names)
        if unknown:
            raise ParseError(f"numeric flag on undeclared fields: {sorted(unknown)}")
        self._ids = {n: i for i, n in enumerate(self.field_names)}

    @property
    def n_fields(self) -> int:
        return len(self.field_names)

    def field_id(self, name: str) -> int:
        from .errors import ParseError
        try:
            return self._ids[name]
        except KeyError:
            raise ParseError(f"unknown field name: {name!r}") from None

    @classmethod
    def from_text(cls, text: str) -> "InputSchema":
        from .errors import ParseError
        names, numeric, hash_bits = [], set(), 18
        for lineno, raw in enumerate(text.splitlines(), 1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.split()
            if parts[0] == "field" and len(parts) in (2, 3):
                if len(parts) == 3 and parts[2] != "numeric":
                    raise ParseError(f"schema line {lineno}: unknown flag {parts[2]!r}")
                names.append(parts[1])
                if len(parts) == 3:
                    numeric.add(parts[1])
            elif parts[0] == "hash_bits" and len(parts) == 2:
                try:
                    hash_bits = int(parts[1])
                except ValueError:
                    raise ParseError(f"schema line {lineno}: hash_bits wants an integer") from None
            else:
                raise ParseError(f"schema line {lineno}: cannot parse {raw!r}")
        return cls(tuple(names), frozenset(numeric), hash_bits)

    def to_text(self) -> str:
        lines = [f"hash_bits {self.hash_bits}"]
        for name in self.field_names:
            lines.append(f"field {name}{' numeric' if name in self.numeric_fields else ''}")
        return "\n".join(lines) + "\n"


class ParsedLines:
    """K10 output on the device: a RaggedBatch of torch tensors plus labels,
    per-line status, the largest per-field count, and optional f64 values."""

    def __init__(self, batch, labels, status, val64=None):
        self.batch, self.labels, self.status, self.val64 = batch, labels, status, val64

    def first_error(self, skip_blank: bool = True):
        """(line number, message) of the first line that failed, or None;
        blank lines (status 11) count only with ``skip_blank=False``."""
        import torch
        bad = torch.nonzero((self.status != 0) & ((self.status != 11) | (not skip_blank)))
        if bad.numel() == 0:
            return None
        i = int(bad[0, 0])
        return i, PARSE_ERRORS.get(int(self.status[i]), "parse error")


def split_lines(text) -> tuple[np.ndarray, np.ndarray]:
    """Bytes of newline-separated lines -> (uint8 buffer, line offsets int64
    [n+1]); line i = buf[off[i]:off[i+1]] keeps its '\n' (trailing whitespace
    to the grammar, Fe:190/Fe:222).  A final line without '\n' counts; nothing
    after the last '\n' does."""
    buf = np.frombuffer(bytes(text), dtype=np.uint8) if not isinstance(text, np.ndarray) \
        else np.ascontiguousarray(text, np.uint8)
    nl = np.flatnonzero(buf == 10) + 1
    ends = nl if (len(buf) == 0 or buf[-1] == 10) else np.append(nl, len(buf))
    return buf, np.concatenate([[0], ends]).astype(np.int64)


def parse_lines(text, schema: InputSchema, device, keep_f64: bool = False,
                raise_on_error: bool = True, skip_blank: bool = True,
                stream=None) -> ParsedLines:
    """K10: parse example lines on the GPU (parse_example, Fe:221-235, for
    every line at once).  ``text`` is bytes (newline-separated lines).  Lines
    are the batch's examples in order; whitespace-only lines get status 11 and
    no features (the stream loops skip them, T:176); with ``raise_on_error``
    the first failed line raises ``ParseError`` like the reference's loop would."""
    import torch

    from . import _lib
    from .errors import ParseError
    dev = torch.device(device)
    buf, off = split_lines(text)
    n = len(off) - 1
    packed = buf
    F = schema.n_fields
    names = b"".join(nm.encode("utf-8") for nm in schema.field_names)
    noff = np.zeros(F + 1, np.int32)
    np.cumsum([len(nm.encode("utf-8")) for nm in schema.field_names], out=noff[1:])
    numeric = np.array([nm in schema.numeric_fields for nm in schema.field_names], np.uint8)
    t_text = torch.from_numpy(packed.copy()).to(dev)
    t_off = torch.from_numpy(off).to(dev)
    t_names = torch.frombuffer(bytearray(names or b"\0"), dtype=torch.uint8).to(dev)
    t_noff = torch.from_numpy(noff).to(dev)
    t_num = torch.from_numpy(numeric).to(dev)
    lib = _lib.lib()
    nbytes = int(off[-1])
    scratch = torch.empty(int(lib.fw_parse_scratch_bytes(n, nbytes)), dtype=torch.uint8,
                          device=dev)
    labels = torch.empty(n, dtype=torch.uint8, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = torch.empty((n, F), dtype=torch.uint8, device=dev)
    ex_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    mx = torch.empty(1, dtype=torch.int32, device=dev)
    cur = torch.cuda.current_stream(dev)
    s = stream if stream is not None else cur
    if s != cur:
        s.wait_stream(cur)  # inputs were uploaded and outputs allocated on `cur`
    _lib.check(lib.fw_parse_lines(t_text.data_ptr(), t_off.data_ptr(), n, nbytes,
                                  t_names.data_ptr(), t_noff.data_ptr(), t_num.data_ptr(), F,
                                  schema.hash_bits, scratch.data_ptr(), labels.data_ptr(),
                                  status.data_ptr(), cnt.data_ptr(), ex_off.data_ptr(),
                                  mx.data_ptr(), s.cuda_stream), "fw_parse_lines")
    s.synchronize()  # the emit pass needs the total; .item() alone syncs only `cur`
    nnz = int(ex_off[n].item())
    idx = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float32, device=dev)
    val64 = torch.empty(nnz, dtype=torch.float64, device=dev) if keep_f64 else None
    if nnz:
        _lib.check(lib.fw_parse_emit(t_off.data_ptr(), n, nbytes, scratch.data_ptr(),
                                     ex_off.data_ptr(), idx.data_ptr(), val.data_ptr(),
                                     val64.data_ptr() if keep_f64 else None, s.cuda_stream),
                   "fw_parse_emit")
    if s != cur:
        cur.wait_stream(s)  # outputs are consumed on the caller's stream
    out = ParsedLines(RaggedBatch(ex_off, cnt, idx, val, max(1, int(mx.item()))), labels,
                      status, val64)
    if raise_on_error:
        err = out.first_error(skip_blank)
        if err is not None:
            raise ParseError(f"line {err[0] + 1}: {err[1]}")
    return out


class HostTextParser:
    """K10 from pinned host text, pipelined: the batch's lines are cut into
    chunks; chunk j+1's text and line offsets travel host->device on a copy
    stream while K10 parses chunk j on one of two compute streams (consecutive
    chunks' parses overlap too), so the link and the parse overlap
    (``parse_lines`` copies the whole text, then parses).

    Each chunk is one ``fw_parse_lines`` + ``fw_parse_emit`` call on global
    pointers: the text window base is relative to the chunk's first line
    (line_off[0]), so chunk-sized scratch suffices and labels/status/cnt land
    at the chunk's global rows.  idx/val of chunk j start at element
    (off[c0] // 2 + c0) of one buffer -- every chunk's capacity (bytes/2 +
    lines) fits below the next chunk's base -- so no host read of a chunk's
    total is needed between chunks.  ``__call__`` returns a ParsedLines per
    chunk (RaggedBatch views) after one synchronise at the end."""

    def __init__(self, schema: InputSchema, device, max_lines: int, max_bytes: int,
                 chunk_lines: int = 1 << 17):
        import torch

        from . import _lib
        self.schema, self.dev = schema, torch.device(device)
        self.chunk = max(1, int(min(chunk_lines, max(1, max_lines))))
        self.max_lines, self.max_bytes = int(max_lines), int(max_bytes)
        F = schema.n_fields
        names = b"".join(nm.encode("utf-8") for nm in schema.field_names)
        noff = np.zeros(F + 1, np.int32)
        np.cumsum([len(nm.encode("utf-8")) for nm in schema.field_names], out=noff[1:])
        numeric = np.array([nm in schema.numeric_fields for nm in schema.field_names], np.uint8)
        dev = self.dev
        self.t_names = torch.frombuffer(bytearray(names or b"\0"), dtype=torch.uint8).to(dev)
        self.t_noff = torch.from_numpy(noff).to(dev)
        self.t_num = torch.from_numpy(numeric).to(dev)
        self.d_text = torch.empty(max(1, self.max_bytes), dtype=torch.uint8, device=dev)
        self.d_off = torch.empty(self.max_lines + 1, dtype=torch.int64, device=dev)
        nchunks_max = (self.max_lines + self.chunk - 1) // self.chunk + 1
        cap = self.max_bytes // 2 + self.max_lines + 1
        self.idx = torch.empty(cap, dtype=torch.int32, device=dev)
        self.val = torch.empty(cap, dtype=torch.float32, device=dev)
        self.labels = torch.empty(max(1, self.max_lines), dtype=torch.uint8, device=dev)
        self.status = torch.empty(max(1, self.max_lines), dtype=torch.int32, device=dev)
        self.cnt = torch.empty((max(1, self.max_lines), F), dtype=torch.uint8, device=dev)
        self.ex_off = torch.empty(self.max_lines + nchunks_max, dtype=torch.int64, device=dev)
        self.mx = torch.empty(nchunks_max, dtype=torch.int32, device=dev)
        self.scratch_cap = 0
        self.scratch = [None, None]
        self.copy_stream = torch.cuda.Stream(dev)
        # two compute streams, alternate chunks: K10 is one thread per line, so one
        # chunk's launches leave most of the machine idle; consecutive chunks overlap
        self.compute_streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        self._lib = _lib

    def _bounds(self, off: np.ndarray):
        n = len(off) - 1
        return [(c0, min(n, c0 + self.chunk)) for c0 in range(0, n, self.chunk)]

    def __call__(self, h_text, h_off, status_host=None):
        """``h_text``: pinned uint8 tensor of the text, ``h_off``: pinned int64
        tensor of line offsets [n+1] (``split_lines``); optional pinned int32
        ``status_host`` [n] receives the per-line status (D2H inside the
        pipeline).  Returns a list of (c0, c1, ParsedLines) per chunk."""
        import torch
        lib = self._lib.lib()
        off = h_off.numpy()
        n = len(off) - 1
        if n > self.max_lines or int(off[-1]) > self.max_bytes:
            raise ContractError(f"{n} lines / {int(off[-1])} bytes exceed the parser's "
                                f"{self.max_lines} / {self.max_bytes}")
        bounds = self._bounds(off)
        need = max((int(lib.fw_parse_scratch_bytes(c1 - c0, int(off[c1] - off[c0])))
                    for c0, c1 in bounds), default=0)
        if need > self.scratch_cap:
            self.scratch = [torch.empty(need, dtype=torch.uint8, device=self.dev)
                            for _ in range(2)]
            self.scratch_cap = need
        cs = self.copy_stream
        cs.wait_stream(torch.cuda.current_stream(self.dev))
        for ks in self.compute_streams:
            ks.wait_stream(cs)
        F = self.schema.n_fields
        evs = []
        for j, (c0, c1) in enumerate(bounds):
            b0, b1 = int(off[c0]), int(off[c1])
            ev = torch.cuda.Event()
            with torch.cuda.stream(cs):
                self.d_text[b0:b1].copy_(h_text[b0:b1], non_blocking=True)
                self.d_off[c0:c1 + 1].copy_(h_off[c0:c1 + 1], non_blocking=True)
                ev.record(cs)
            evs.append(ev)
            base = b0 // 2 + c0
            eo = self.ex_off[c0 + j:c1 + j + 1]
            ks, scr = self.compute_streams[j & 1], self.scratch[j & 1]
            with torch.cuda.stream(ks):
                ks.wait_event(ev)
                self._lib.check(lib.fw_parse_lines(
                    self.d_text.data_ptr(), self.d_off[c0:].data_ptr(), c1 - c0, b1 - b0,
                    self.t_names.data_ptr(), self.t_noff.data_ptr(), self.t_num.data_ptr(), F,
                    self.schema.hash_bits, scr.data_ptr(),
                    self.labels[c0:].data_ptr(), self.status[c0:].data_ptr(),
                    self.cnt[c0:].data_ptr(), eo.data_ptr(), self.mx[j:].data_ptr(),
                    ks.cuda_stream), "fw_parse_lines")
                self._lib.check(lib.fw_parse_emit(
                    self.d_off[c0:].data_ptr(), c1 - c0, b1 - b0, scr.data_ptr(),
                    eo.data_ptr(), self.idx[base:].data_ptr(), self.val[base:].data_ptr(),
                    None, ks.cuda_stream), "fw_parse_emit")
                if status_host is not None:
                    status_host[c0:c1].copy_(self.status[c0:c1], non_blocking=True)
        ks = self.compute_streams[0]
        ks.wait_stream(self.compute_streams[1])
        with torch.cuda.stream(ks):
            ends = torch.tensor([c1 + j for j, (_, c1) in enumerate(bounds)], dtype=torch.int64,
                                device=self.dev) if bounds else None
            tail = (torch.stack([self.ex_off[ends], self.mx[:len(bounds)].to(torch.int64)])
                    .cpu() if bounds else None)
        ks.synchronize()
        out = []
        for j, (c0, c1) in enumerate(bounds):
            nnz, mxc = int(tail[0, j]), int(tail[1, j])
            base = int(off[c0]) // 2 + c0
            rb = RaggedBatch(self.ex_off[c0 + j:c1 + j + 1], self.cnt[c0:c1],
                             self.idx[base:base + nnz], self.val[base:base + nnz], max(1, mxc))
            out.append((c0, c1, ParsedLines(rb, self.labels[c0:c1], self.status[c0:c1])))
        return out


def _segment_field_order(line: str, schema: InputSchema):
    """Field ids in order of first appearance (Fe:186-196): the '|' segment heads."""
    order, seen = [], set()
    for seg in line.split("|")[1:]:
        atoms = seg.split()
        if atoms:
            fid = schema.field_id(atoms[0])
            if fid not in seen:
                seen.add(fid)
                order.append(fid)
    return order


def _examples_from_parsed(out: "ParsedLines", lines, schema: InputSchema):
    """K10 output (ragged, f64 values kept) -> ParsedExample per line."""
    b = out.batch
    ex_off = b.ex_off.cpu().numpy()
    cnt = b.cnt.cpu().numpy()
    idx = b.idx.cpu().numpy().astype(np.int64)
    val = out.val64.cpu().numpy()
    labels = out.labels.cpu().numpy()
    res = []
    for i, line in enumerate(lines):
        pos = int(ex_off[i])
        per = {}
        for f in range(schema.n_fields):
            m = int(cnt[i, f])
            if m:
                per[f] = (idx[pos:pos + m].copy(), val[pos:pos + m].copy())
                pos += m
        fields = []
        for f in _segment_field_order(line, schema):
            ii, vv = per.get(f, (np.empty(0, np.int64), np.empty(0, np.float64)))
            fields.append(FieldFeatures(f, ii, vv))
        res.append(ParsedExample(int(labels[i]), tuple(fields)))
    return res


def _check_gpu_status(out: "ParsedLines", first_line: int = 0):
    from .errors import ParseError
    err = out.first_error(skip_blank=False)
    if err is not None:
        i, msg = err
        code = int(out.status[i])
        if code in (8, 9, 10):  # lines the reference accepts but K10 cannot take
            raise ContractError(f"line {first_line + i + 1}: {msg}")
        raise ParseError(f"line {first_line + i + 1}: {msg}")


def parse_example(line: str, schema: InputSchema, device=None) -> ParsedExample:
    """Parse one text example (Fe:223-235) with K10 on the device: label, field
    blocks, FNV-1a hashing, numeric transform, duplicate merge; values kept in
    f64.  Raises ParseError exactly where the reference does."""
    import torch
    dev = torch.device(device) if device is not None else torch.device("cuda")
    text = line.encode("utf-8")
    if b"\n" in text.rstrip(b"\n"):
        from .errors import ParseError
        raise ParseError("one example per line")
    out = parse_lines(text.rstrip(b"\n") + b"\n", schema, dev, keep_f64=True,
                      raise_on_error=False, skip_blank=False)
    if int(out.status[0]) == 11:  # whitespace-only: the reference's label check fails
        from .errors import ParseError
        raise ParseError(f"malformed label {line.split('|')[0].strip()!r} (want 0, 1, or -1)")
    _check_gpu_status(out)
    return _examples_from_parsed(out, [line], schema)[0]


def parse_field_blocks(text: str, schema: InputSchema, device=None) -> tuple:
    """Label-less '|field ...' request text -> FieldFeatures (Fe:238-249)."""
    from .errors import ParseError
    stripped = text.strip()
    if not stripped.startswith("|"):
        raise ParseError("field blocks must start with '|'")
    if stripped == "|":
        return ()
    return parse_example("0 " + stripped, schema, device).fields


def serialize_example(example: ParsedExample, schema: InputSchema) -> str:
    """Debug serializer (Fe:252-264): raw '@index:value' tokens that re-parse
    to an identical ParsedExample."""
    parts = [str(example.label)]
    for ff in example.fields:
        block = [f"|{schema.field_names[ff.field_id]}"]
        for i, v in zip(ff.indices, ff.values):
            block.append(f"@{int(i)}:{float(v)!r}")
        parts.append(" ".join(block))
    return " ".join(parts)
