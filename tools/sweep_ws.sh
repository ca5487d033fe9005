#!/bin/bash
# A/B: K1 v3 (ws) gather-warp counts vs v1 (mb4 build) on cfg2.
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(f\"{d['value']/1e6:.1f}M/s frac={d['roofline']['frac']:.3f} e2e={d['e2e']['value']/1e6:.1f}M/s\")"; }
echo "ws NG=20: $(run)"
for ng in 16 28; do echo "ws NG=$ng: $(DFFM_LIB_PATH=$PWD/tools/libdffm_ng$ng.so run)"; done
echo "v1 mb4 TE16: $(DFFM_FORWARD_KERNEL=v1 DFFM_LIB_PATH=$PWD/tools/libdffm_mb4.so run)"
