#!/bin/bash
# A/B: K1 v3 (ws) gather-warp counts on cfg2, two repetitions each.
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(f\"{d['value']/1e6:.1f}M/s frac={d['roofline']['frac']:.3f} e2e={d['e2e']['value']/1e6:.1f}M/s\")"; }
for rep in 1 2; do
echo "ws NG=16: $(run)"
echo "ws NG=12: $(DFFM_LIB_PATH=$PWD/tools/libdffm_ng12.so run)"
done
