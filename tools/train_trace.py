"""Per-phase K2 latency breakdown from a -DDFFM_TR_TRACE build
(tools/libdffm_trace.so): SM cycles between phase boundaries of thread 0,
averaged over 64 examples of a cfg3-shaped stream."""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("DFFM_LIB_PATH", "tools/libdffm_trace.so")
sys.argv = [sys.argv[0], "400"] + sys.argv[1:]
sys.path.insert(0, ".")
exec(open("tools/train_profile.py").read())  # runs 200 warm-up + 400 examples
from paper_2407_10115_b200 import _lib  # noqa: E402

h = _lib.lib()
NPH = 40
buf = (ctypes.c_longlong * (64 * NPH))()
h.dffm_tr_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(64, NPH)
names = ["start", "staged", "S+lr loaded", "dup lists", "pairs+norm", "mlp l0 fwd", "mlp l1 fwd",
         "mlp out", "bwd l>0", "bwd l0", "norm bwd", "dp/fact", "ffm upd", "lr upd", "cl.sync"]
per = np.median(np.diff(t[:, :15], axis=1), axis=0)
tot = np.median(t[1:, 0] - t[:-1, 0])
for i, d in enumerate(per):
    print(f"{names[i]:>12s} -> {names[i+1]:<12s} {d:8.0f} cyc")
print(f"example period {tot:.0f} cycles")

fine = [(1, 30, "staged -> field warp 1 starts its loads"), (30, 31, "field warp 1: loads issued"),
        (31, 37, "field warp 1: loads landed, sums, S stores"), (1, 36, "staged -> spare warps: dup lists done"), (1, 37, "staged -> field warp 1: S written"),
        (1, 38, "staged -> field warp 0: lr partials + S written"), (1, 3, "staged -> barrier passed"),
        (3, 16, "pairs loop"), (16, 17, "lr_out by thread 0"), (17, 18, "block_sum(pairs)"), (18, 19, "syncthreads_or"),
        (19, 20, "mu, var block_sum, sqrt"), (20, 4, "merged[] + syncthreads_or"), (7, 21, "logit, prefetch"),
        (21, 22, "sigmoid"), (22, 23, "g -> dg, sync"), (23, 26, "out layer upstream + sync"),
        (26, 25, "l1 upstream + sync"), (25, 24, "l0 upstream + cluster reduce + sync"),
        (8, 9, "all MLP updates (thread 0)")]
for a, b, nm in fine:
    d = np.median(t[:, b] - t[:, a])
    print(f"{nm:>34s} {d:8.0f} cyc")
