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

import numpy as np

from .errors import ContractError


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
