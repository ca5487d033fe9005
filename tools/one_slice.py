"""One cfg2 or cfg5 forward slice inside an NVTX range "step" (ncu target).
    python tools/one_slice.py cfg5 [n]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.model import predict_batch  # noqa: E402

wl = {"cfg2": configs.CFG2, "cfg5": configs.CFG5}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 606208
dev = torch.device("cuda", 0)
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
prob = torch.empty(n, device=dev)
for _ in range(2):
    predict_batch(idx, val, st, out=prob, check=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
predict_batch(idx, val, st, out=prob, check=False)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done", n)
