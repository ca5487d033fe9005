"""One cfg4 context-cached scoring step (2,000 requests x 500 candidates, u16 tables)
inside an NVTX range "step" (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_10115_b200 import configs, synth  # noqa: E402
from paper_2407_10115_b200.inference import score_requests  # noqa: E402

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
for _ in range(2):
    score_requests(ci, cv, di, dv, st, out=out, check=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
score_requests(ci, cv, di, dv, st, out=out, check=False)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
