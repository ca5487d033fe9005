"""Quick K1 check on one GPU: per-kernel device time (gather / MLP) of a forward
step and the max relative error against the oracle on a sample, for cfg2 and
cfg5-shaped batches (n examples each).

    python tools/mlp_quick.py [n] [steps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.model import predict_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 606208
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
for wl in (configs.CFG2, configs.CFG5):
    st = bench.build_store(wl, dev)
    idx, val = bench.build_inputs(wl, n, dev, 0)
    prob = torch.empty(n, device=dev)
    flush = torch.empty(64 << 20, device=dev)
    for _ in range(3):
        predict_batch(idx, val, st, out=prob, check=False)
    torch.cuda.synchronize()
    tr = bench.LaunchTrace(per_step=64, steps=steps)
    with tr:
        for _ in range(steps):
            flush.zero_()
            s = torch.cuda.Event(enable_timing=True)
            s.record()
            tr.mark_step(s)
            predict_batch(idx, val, st, out=prob, check=False)
        torch.cuda.synchronize()
    split = {k: round(v[0] / steps, 3) for k, v in tr.split().items()}
    try:
        predict_batch(idx, val, st, out=prob, check=True)
    except Exception as exc:  # measurement variants produce garbage on purpose
        print(f"{wl.name}: n={n} ms/step {split}  (check failed: {type(exc).__name__})",
              flush=True)
        del st, idx, val, prob
        torch.cuda.empty_cache()
        continue
    m = 2048
    ost, ridx = bench.compact_oracle_store(st, idx[:m].cpu().numpy())
    ref, _ = bench.run_cpu_port(ost, ridx, val[:m].cpu().numpy(), 8)
    err = float(np.max(np.abs(prob[:m].double().cpu().numpy() - ref) / ref))
    print(f"{wl.name}: n={n} ms/step {split}  max rel err {err:.3e}", flush=True)
    del st, idx, val, prob
    torch.cuda.empty_cache()
