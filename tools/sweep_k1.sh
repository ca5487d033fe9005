#!/bin/bash
# A/B sweep of K1 v1 build variants (min blocks/SM) x tile width on cfg2.
export DFFM_FORWARD_KERNEL=v1
for lib in default mb3 mb4; do
  for te in 8 16 32; do
    if [ $lib = default ]; then unset DFFM_LIB_PATH; else export DFFM_LIB_PATH=$PWD/tools/libdffm_$lib.so; fi
    v=$(DFFM_FWD_TE=$te timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(f\"{d['value']/1e6:.1f}M/s {d['roofline']['frac']:.3f} e2e {d['e2e']['value']/1e6:.1f}M/s\")")
    echo "lib=$lib TE=$te $v"
  done
done
