"""cfg2 / cfg5 forward over n examples: ms per forward (CUDA events, L2 flushed between
forwards) with the gather / MLP split from the library's event trace.  A/B tool: select the
library with DFFM_LIB_PATH.   python tools/fwd_quick.py cfg5 [n] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.model import predict_batch  # noqa: E402

wl = {"cfg2": configs.CFG2, "cfg5": configs.CFG5}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1048576 if wl is configs.CFG2 else 4 * 606208)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
dev = torch.device("cuda", 0)
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
prob = torch.empty(n, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    predict_batch(idx, val, st, out=prob, check=False)
torch.cuda.synchronize()
ms = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    predict_batch(idx, val, st, out=prob, check=False)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
ms.sort()
m = ms[len(ms) // 2]
print(f"{wl.name} n={n}: median {m:.3f} ms  min {ms[0]:.3f}  -> {n / m / 1e3:.1f} M preds/s  "
      f"checksum {prob.double().sum().item():.6f}")
