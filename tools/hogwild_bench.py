"""K6 scaling on cfg3 (2^24 buckets, teacher-planted labels): examples/s and
progressive logloss vs workers (N=1 = the exact sequential kernel)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_10115_b200 import configs, synth  # noqa: E402
from paper_2407_10115_b200.model import ModelConfig, WeightStore, predict_batch  # noqa: E402
from paper_2407_10115_b200.training import (TrainOptions, hogwild_train_arrays,  # noqa: E402
                                             max_hogwild_workers)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
wl = configs.CFG3
dev = torch.device("cuda:0")
cfg = ModelConfig(n_fields=24, k=8, hidden_sizes=(64, 32), hash_bits=24, lr_ffm=0.1, lr_lr=0.1,
                  lr_nn=0.1)
idx, val = synth.make_examples(wl, n, device=dev)


def store(seed):
    st = WeightStore(cfg, dev, with_optimizer=True).fill_accumulators(1.0)
    g = torch.Generator(device=dev).manual_seed(seed)
    for t in [st.lr, st.ffm] + [x for wb in st.nn_layers for x in wb]:
        flat = t.view(-1)
        for c0 in range(0, flat.numel(), 1 << 28):
            c1 = min(flat.numel(), c0 + (1 << 28))
            flat[c0:c1].copy_(torch.randn(c1 - c0, generator=g, device=dev) * 0.05)
    return st


teacher = store(3003)
p = predict_batch(idx, val, teacher)
labels = (torch.rand(n, generator=torch.Generator(device=dev).manual_seed(7), device=dev) < p).to(torch.uint8)
del teacher
torch.cuda.empty_cache()
wmax = max_hogwild_workers(store(1), idx.shape[2])
print(f"max concurrent workers: {wmax}")
for w in [1, 4, 16, 64, 148, wmax]:
    st = store(1004)
    m = n if w > 1 else min(n, 50000)
    hogwild_train_arrays(idx[:200], val[:200], labels[:200], st, TrainOptions(n_threads=w))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = hogwild_train_arrays(idx[200:m], val[200:m], labels[200:m], st, TrainOptions(n_threads=w))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"workers={w:4d} examples={m - 200} ex/s={(m - 200) / dt:12.0f} "
          f"progressive_logloss={rep.progressive_logloss:.5f}")
    del st
    torch.cuda.empty_cache()
