"""Timeline of the tcgen05 MLP's MMA issuer on CTA 0 (variant build with
-DDFFM_TC_TRACE): per tile, cycles spent waiting for the first chunk of each
layer and issuing it.  DFFM_LIB_PATH=build_var/tct/libdffm.so python tools/tc_trace.py cfg5"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import _lib, configs  # noqa: E402
from paper_2407_10115_b200.model import predict_batch  # noqa: E402

wl = {"cfg2": configs.CFG2, "cfg5": configs.CFG5}[sys.argv[1]]
n = 606208
dev = torch.device("cuda", 0)
st = bench.build_store(wl, dev)
idx, val = bench.build_inputs(wl, n, dev, 0)
prob = torch.empty(n, device=dev)
predict_batch(idx, val, st, out=prob, check=False)
torch.cuda.synchronize()
fn = _lib.lib().dffm_debug_tc_trace
fn.restype = ctypes.c_int
buf = (ctypes.c_longlong * 4096)()
fn(buf, 4096)  # reset
predict_batch(idx, val, st, out=prob, check=False)
torch.cuda.synchronize()
k = fn(buf, 4096)
ev = [(v >> 8, v & 0xFF) for v in buf[:k]]
t0 = ev[0][0]
rows = []
cur = {}
for t, tag in ev:
    cur[tag] = t - t0
    if tag == 17:  # end of layer 1 issue = end of a tile
        rows.append(dict(cur))
        cur = {}
print("tiles", len(rows))
keys = [0, 1, 16, 2, 3, 17]
names = {0: "L0 wait-start", 1: "L0 first full", 16: "L0 issued", 2: "L1 wait-start",
         3: "L1 first full", 17: "L1 issued"}
d = np.array([[r.get(kk, 0) for kk in keys] for r in rows], dtype=np.float64)
tile = np.diff(d[:, 5])
print("cycles per tile (median)", np.median(tile))
print("L0: first chunk wait", np.median(d[:, 1] - d[:, 0]), " issue of all L0 chunks",
      np.median(d[:, 2] - d[:, 1]))
print("L0 end -> L1 first full (wait aready/full)", np.median(d[:, 4] - d[:, 2]),
      " L1 issue", np.median(d[:, 5] - d[:, 4]))
print("L1 end -> next L0 first full", np.median(d[1:, 1] - d[:-1, 5]))
# epilogue stamps (warp 2 lane 0): per tile, relative to the MMA's L0 issue end
evs = sorted(ev)
tl = [t for t, tag in evs if tag == 16]
def after(tag, t0):
    xs = [t for t, g in evs if g == tag and t >= t0]
    return xs[0] - t0 if xs else float("nan")
for tag, nm in [(32, "epi at last L0 drain"), (40, "epi L0 drained"), (48, "epi bias/relu done"),
                (56, "epi exchange barrier passed"), (64, "epi A1 written+arrived"),
                (3, "MMA L1 first full")]:
    print(f"  {nm:30s} +{np.nanmedian([after(tag, t) for t in tl[1:-1]]):.0f} after L0 issue end")
