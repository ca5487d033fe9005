"""cfg3 at full size: n-example prefix on the GPU vs the oracle on the remapped touched
rows; prints how many touched slots are outside |dw| <= 1e-5 max(|w|, 1e-3) and by how
much (the slow parity test's criterion, with statistics).  DFFM_LIB_PATH selects the
library; OLD_CDF=1 sums the Zipf CDF on the device as before round 2's synth change."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import fieldwise_oracle as fo  # noqa: E402
from paper_2407_10115_b200 import configs, synth  # noqa: E402
from paper_2407_10115_b200.model import ModelConfig, WeightStore  # noqa: E402
from paper_2407_10115_b200.training import train_sequential  # noqa: E402
from tests.remap import compact_oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 120000
DEV = torch.device("cuda:0")
if os.environ.get("OLD_CDF"):
    def _cdf(nn, alpha, device):
        r = torch.arange(1, nn + 1, dtype=torch.float64, device=device)
        c = torch.cumsum(r.pow(-alpha), 0)
        return c / c[-1]
    synth.zipf_cdf = _cdf
wl = configs.CFG3
cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=24, lr_ffm=0.1, lr_lr=0.1,
                  lr_nn=0.1, power_t=0.5)
st = WeightStore(cfg, DEV).fill_accumulators(1.0)
gen = torch.Generator(device=DEV).manual_seed(wl.weight_seed)
st.lr.copy_(synth.normal_table(st.lr.numel(), 0.05, gen, DEV))
st.ffm.view(-1).copy_(synth.normal_table(st.ffm.numel(), 0.05, gen, DEV))
for w, b in st.nn_layers:
    w.copy_(torch.randn(w.shape, generator=gen, device=DEV) * 0.05)
    b.copy_(torch.randn(b.shape, generator=gen, device=DEV) * 0.05)
idx, val = synth.make_examples(wl, n, device=DEV)
labels = synth.make_labels(n, 0.3, 5, device=DEV)
ih, vh, lh = idx.cpu().numpy(), val.cpu().numpy(), labels.cpu().numpy()
ost, ridx, u = compact_oracle(st, ih)
rep = train_sequential(idx, val, labels, st)
probs, _ = fo.train_sequential(ridx, vh, lh, ost, .1, .1, .1, .5)
rel = np.abs(rep.probs - probs) / probs
first = int(np.argmax(rel > 1e-9)) if (rel > 1e-9).any() else -1
print(f"probs: max rel err {rel.max():.3e}; first example with rel err > 1e-9: {first}; "
      f"rel err at 1k/10k/50k/last: {rel[1000]:.2e} {rel[min(10000, n-1)]:.2e} {rel[min(50000, n-1)]:.2e} {rel[-1]:.2e}")
ut = torch.as_tensor(u, device=DEV)
got = np.concatenate([st.ffm[ut].cpu().numpy().ravel(), st.ffm_acc[ut].cpu().numpy().ravel(),
                      st.lr[ut].cpu().numpy(), st.lr_acc[ut].cpu().numpy()])
ref = np.concatenate([ost.ffm[:len(u)].ravel(), ost.ffm_acc[:len(u)].ravel(), ost.lr[:len(u)],
                      ost.lr_acc[:len(u)]])
tol = 1e-5 * np.maximum(np.abs(ref), 1e-3)
d = np.abs(got.astype(np.float64) - ref)
bad = d > tol
print(f"touched slots {got.size}: outside tolerance {int(bad.sum())}, bit-identical {np.mean(got == ref):.4%}, "
      f"max |d|/tol {np.max(d / tol):.3f}, 99.99th pct {np.quantile(d / tol, 0.9999):.3f}")
if (rel > 1e-12).any():
    e0 = int(np.argmax(rel > 1e-12))
    print("first example with rel err > 1e-12:", e0, "rel", rel[e0])
    rows_e0 = set(ih[e0][ih[e0] >= 0].tolist())
    # the most recent earlier examples that share a bucket with e0
    cand = []
    for e in range(e0 - 1, max(-1, e0 - 200000), -1):
        sh = rows_e0 & set(ih[e][ih[e] >= 0].tolist())
        if sh:
            cand.append((e, len(sh)))
        if len(cand) >= 6:
            break
    print("recent examples sharing buckets with it:", cand)
    for e in [e0] + [c[0] for c in cand[:3]]:
        live = ih[e][ih[e] >= 0]
        uq, cnt = np.unique(live, return_counts=True)
        print(f"example {e}: slots {live.size}, unique buckets {uq.size}, duplicated buckets {uq[cnt > 1].tolist()}, "
              f"val min {vh[e][ih[e] >= 0].min():.4g} max {vh[e][ih[e] >= 0].max():.4g}, label {lh[e]}, "
              f"gpu p {rep.probs[e]:.12g} oracle p {probs[e]:.12g}")
        if (cnt > 1).any():
            for b in uq[cnt > 1]:
                pos = np.argwhere(ih[e] == b)
                print("   bucket", int(b), "at (field, slot):", pos.tolist(), "vals", [float(vh[e][tuple(p)]) for p in pos])
