"""Sweep HostPredictor chunk sizes for the padded and ragged e2e paths (cfg2)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.features import PackedBatch, RaggedBatch  # noqa: E402
from paper_2407_10115_b200.model import HostPredictor  # noqa: E402

dev = torch.device("cuda:0")
wl = configs.CFG2
n = wl.n_examples
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
idx_h, val_h = idx.cpu().pin_memory(), val.cpu().pin_memory()
rb = RaggedBatch.from_padded(idx_h.numpy(), val_h.numpy())
rbh = RaggedBatch(*(torch.from_numpy(a).pin_memory() for a in (rb.ex_off, rb.cnt, rb.idx, rb.val)),
                  rb.max_per_field)
pk = PackedBatch.from_ragged(rb)
pin = lambda a: torch.from_numpy(a.copy()).pin_memory()  # noqa: E731
pkh = PackedBatch(pin(pk.ex_off), pin(pk.cnt), pin(pk.idx_bytes), pk.idx_width, pin(pk.vbits),
                  pin(pk.vals), pin(pk.voff), pk.max_per_field)
out = torch.empty(n, dtype=torch.float32).pin_memory()
for ch in [1 << 17, 1 << 18, 1 << 19]:
    hp = HostPredictor(st, n, idx.shape[2], chunk=ch)
    for name, fn in [("ragged", lambda: hp.predict_ragged(rbh, out)),
                     ("packed", lambda: hp.predict_packed(pkh, out))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        dt = (time.perf_counter() - t0) / 5
        print(f"chunk {ch:7d} {name}: {n / dt / 1e6:7.2f} M preds/s", flush=True)
