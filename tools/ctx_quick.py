"""cfg4 context-cached scoring (2,000 requests x 500 candidates, u16 tables): ms per
step over N steps (CUDA events, L2 flushed between steps).  A/B tool: select the
library with DFFM_LIB_PATH, knobs with DFFM_CTX_*."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs, synth  # noqa: E402
from paper_2407_10115_b200.inference import score_requests  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
wl = configs.CFG4
dev = torch.device("cuda", 0)
R, C, Fc, F = wl.n_requests, wl.n_candidates, wl.ctx_fields, wl.n_fields
st = bench.build_store(wl, dev)
cdf = synth.zipf_cdf(1 << wl.hash_bits, wl.zipf_alpha, dev)
ci, cv = synth.make_examples(wl, R, seed=wl.data_seed, device=dev, cdf=cdf, n_fields=Fc)
di, dv = synth.make_examples(wl, R * C, seed=wl.data_seed + 1, device=dev, cdf=cdf,
                             n_fields=F - Fc, field_offset=Fc)
di, dv = di.view(R, C, F - Fc, -1), dv.view(R, C, F - Fc, -1)
out = torch.empty((R, C), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    score_requests(ci, cv, di, dv, st, out=out, check=False)
torch.cuda.synchronize()
ms = []
for _ in range(steps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    score_requests(ci, cv, di, dv, st, out=out, check=False)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
ms.sort()
print(f"cfg4 median {ms[len(ms)//2]:.3f} ms  min {ms[0]:.3f}  -> {R*C/ms[len(ms)//2]/1e3:.1f} M cand/s  "
      f"checksum {out.double().sum().item():.6f}")
