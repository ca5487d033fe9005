"""Run K2 on a cfg3-shaped prefix (for ncu / timing)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_10115_b200 import configs, synth  # noqa: E402
from paper_2407_10115_b200.model import ModelConfig, WeightStore  # noqa: E402
from paper_2407_10115_b200.training import TrainOptions, train_sequential  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 24
wl = configs.CFG3
dev = torch.device("cuda:0")
cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=bits, lr_ffm=0.1, lr_lr=0.1,
                  lr_nn=0.1)
st = WeightStore(cfg, dev).fill_accumulators(1.0)
g = torch.Generator(device=dev).manual_seed(1)
for t in [st.lr, st.ffm] + [x for wb in st.nn_layers for x in wb]:
    t.view(-1).copy_(torch.randn(t.numel(), generator=g, device=dev) * 0.05)
idx, val = synth.make_examples(wl, n, device=dev, hash_bits=bits)
labels = synth.make_labels(n, 0.3, 5, device=dev)
train_sequential(idx[:200], val[:200], labels[:200], st)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = train_sequential(idx, val, labels, st)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{n} examples in {dt:.3f}s -> {n/dt:.0f} ex/s, {1e6*dt/n:.1f} us/example")
