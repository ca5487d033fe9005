#!/bin/bash
# A/B: K1 v5 (gather4) smem caps / tile widths vs v3 (ws) on cfg2.
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --train-examples 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"{d['value']/1e6:.1f}M/s frac={d['roofline']['frac']:.3f} e2e={d['e2e']['value']/1e6:.1f}M/s\")" 2>&1 | tail -1; }
echo "ws: $(DFFM_FORWARD_KERNEL=ws run)"
for kb in 120 160 200 227; do for te in 16 32; do
  echo "g4 smem=${kb}KB TE=$te: $(DFFM_FORWARD_KERNEL=g4 DFFM_G4_SMEM_KB=$kb DFFM_G4_TE=$te run)"
done; done
