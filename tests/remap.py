"""Monotone index-remap oracle: run the CPU oracle on the rows a
parity sample touches, copied back from a full-size device store."""

import math

import numpy as np
import torch

from oracle import fieldwise_oracle as fo


def compact_oracle(store, idx, extra_idx=None):
    """(OracleStore over the touched rows, remapped idx) for a device store.

    Buckets are mapped to 0..U-1 in sorted order; the bias keeps its slot at
    the compact store's own 2^b.  Values are the device tables' f32 values
    (bf16 / u16 tables are widened / dequantised exactly as K1 does)."""
    idx = np.asarray(idx)
    allidx = idx if extra_idx is None else np.concatenate([idx.ravel(), np.asarray(extra_idx).ravel()])
    u = np.unique(allidx[allidx >= 0])
    bits = max(1, math.ceil(math.log2(max(len(u), 2))))
    cfg = store.config
    ost = fo.OracleStore.zeros(cfg.n_fields, cfg.k, cfg.hidden_sizes, bits)
    ut = torch.as_tensor(u, dtype=torch.int64, device=store.device)
    if store.wdtype == "u16":
        from paper_2407_10115_b200.quant import dequantize_tensor, take_rows
        hl, bl = store.q_headers["lr"]
        hf, bf = store.q_headers["ffm"]
        lr_rows = dequantize_tensor(take_rows(store.lr, ut), hl, bl).cpu().numpy()
        bias = dequantize_tensor(take_rows(store.lr, ut[-1:] * 0 + store.n_features), hl, bl).cpu().numpy()[0]
        ffm_rows = dequantize_tensor(take_rows(store.ffm, ut), hf, bf).cpu().numpy()
    else:
        lr_rows = store.lr[ut].float().cpu().numpy()
        bias = store.lr[-1].float().item()
        ffm_rows = store.ffm[ut].float().cpu().numpy()
    ost.lr[: len(u)] = lr_rows
    ost.lr[ost.n_features] = bias
    ost.ffm[: len(u)] = ffm_rows
    for i, (w, b) in enumerate(store.nn_layers):
        ost.layers[i][0][:] = w.float().cpu().numpy()
        ost.layers[i][1][:] = b.float().cpu().numpy()
    if store.has_optimizer:
        ost.lr_acc[: len(u)] = store.lr_acc[ut].cpu().numpy()
        ost.lr_acc[ost.n_features] = store.lr_acc[-1].item()
        ost.ffm_acc[: len(u)] = store.ffm_acc[ut].cpu().numpy()
        for i, (w, b) in enumerate(store.nn_accs):
            ost.layer_accs[i][0][:] = w.cpu().numpy()
            ost.layer_accs[i][1][:] = b.cpu().numpy()
    remapped = np.where(idx >= 0, np.searchsorted(u, np.maximum(idx, 0)), -1).astype(np.int32)
    return ost, remapped, u


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
