"""Run the same forward several times in one process and compare the probabilities bit
for bit (race detector for the warp-specialised gather / tcgen05 MLP)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs  # noqa: E402
from paper_2407_10115_b200.model import predict_batch  # noqa: E402

wl = {"cfg2": configs.CFG2, "cfg5": configs.CFG5}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2 * 606208
dev = torch.device("cuda", 0)
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
ref = predict_batch(idx, val, st, check=True).clone()
print("checksum", ref.double().sum().item(), "inputs", int(idx.long().sum().item()), float(val.double().sum().item()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for r in range(8):
    if r & 1:
        flush.zero_()
    p = predict_batch(idx, val, st, check=False)
    torch.cuda.synchronize()
    d = (p != ref).nonzero().flatten()
    if d.numel():
        i = int(d[0])
        print(f"run {r}: {d.numel()} examples differ; first {i}: {ref[i].item():.9f} vs {p[i].item():.9f}; "
              f"max abs diff {(p - ref).abs().max().item():.3e}")
    else:
        print(f"run {r}: identical")
