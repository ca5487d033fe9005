import sys, time
import torch
sys.path.insert(0, ".")
import bench
from paper_2407_10115_b200 import configs
from paper_2407_10115_b200.model import predict_batch
dev = torch.device("cuda:0")
wl = configs.CFG2; n = wl.n_examples
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
prob = torch.empty(n, device=dev)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
full = timeit(lambda: predict_batch(idx, val, st, out=prob, check=False))
print("kernel 1M one launch: %.2f ms" % (full * 1e3))
for ch in [1 << 16, 1 << 17]:
    def chunked():
        for c0 in range(0, n, ch):
            predict_batch(idx[c0:c0+ch], val[c0:c0+ch], st, out=prob[c0:c0+ch], check=False)
    print("kernel chunked %d: %.2f ms" % (ch, timeit(chunked) * 1e3))
idx_h = idx.cpu().pin_memory(); val_h = val.cpu().pin_memory()
d_i = torch.empty_like(idx); d_v = torch.empty_like(val)
def h2d():
    d_i.copy_(idx_h, non_blocking=True); d_v.copy_(val_h, non_blocking=True)
t = timeit(h2d)
print("H2D padded 604MB: %.2f ms = %.1f GB/s" % (t * 1e3, 604e6 / t / 1e9))
