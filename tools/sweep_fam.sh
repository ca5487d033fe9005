#!/bin/bash
# A/B: K1 kernel families on cfg2 (two repetitions).
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(f\"{d['value']/1e6:.1f}M/s frac={d['roofline']['frac']:.3f} e2e={d['e2e']['value']/1e6:.1f}M/s\")"; }
for rep in 1 2; do
  for te in 16 32; do echo "rows TE=$te: $(DFFM_ROWS_TE=$te run)"; done
  echo "ws: $(DFFM_FORWARD_KERNEL=ws run)"
done
