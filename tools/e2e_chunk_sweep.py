"""Sweep HostPredictor's chunk size for the e2e host-buffer paths (cfg2).

Run on the GPU box: python tools/e2e_chunk_sweep.py
Prints examples/s per (format, chunk); each point is the mean of 5 calls after 1 warm-up,
timed by wall clock around the synchronous call (as bench.py's e2e)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.features import PackedBatch, RaggedBatch  # noqa: E402
from paper_2407_10115_b200.model import HostPredictor, predict_batch  # noqa: E402


def main():
    wl = configs.CFG2
    dev = torch.device("cuda", 0)
    n = wl.n_examples
    st = bench.build_store(wl, dev)
    idx, val = bench.build_inputs(wl, n, dev, 0)
    prob = torch.empty(n, dtype=torch.float32, device=dev)
    predict_batch(idx, val, st, out=prob, check=True)
    prob_h = prob.cpu()
    idx_h, val_h = idx.cpu().pin_memory(), val.cpu().pin_memory()
    rb = RaggedBatch.from_padded(idx_h.numpy(), val_h.numpy())
    rb_h = RaggedBatch(*(torch.from_numpy(a).pin_memory() for a in (rb.ex_off, rb.cnt, rb.idx,
                                                                    rb.val)), rb.max_per_field)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    pk = PackedBatch.from_ragged(rb)
    pk_h = PackedBatch(pin(pk.ex_off), pin(pk.cnt), pin(pk.idx_bytes), pk.idx_width,
                       pin(pk.vbits), pin(pk.vals), pin(pk.voff), pk.max_per_field)
    out_h = torch.empty(n, dtype=torch.float32).pin_memory()
    for chunk in (1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20):
        hp = HostPredictor(st, n, idx.shape[2], chunk=chunk)
        for name, fn in (("padded", lambda: hp(idx_h, val_h, out_h)),
                         ("ragged", lambda: hp.predict_ragged(rb_h, out_h)),
                         ("packed", lambda: hp.predict_packed(pk_h, out_h))):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                fn()
            dt = (time.perf_counter() - t0) / 5
            ok = bool(torch.equal(out_h, prob_h))
            print(f"chunk={chunk:>8} {name:>7}: {n / dt / 1e6:7.1f} M preds/s  match={ok}",
                  flush=True)
        del hp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
