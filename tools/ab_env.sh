#!/bin/bash
# A/B one env knob on cfg5 (default path) and cfg2 (tc path):  tools/ab_env.sh VAR "v1 v2 ..."
set -u
OUT=gpurun_out/ab; mkdir -p $OUT
VAR=$1; VALS=$2
B5="python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --train-examples 0"
B2="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --train-examples 0"
show() { python -c "import json; d=json.load(open('$1')); print('$1', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -n 3 ${1%.json}.err; }
for v in $VALS; do
  export $VAR=$v
  timeout 300 $B5 > $OUT/e5_$v.json 2> $OUT/e5_$v.err; show $OUT/e5_$v.json
  [ -z "${SKIP2:-}" ] && { DFFM_FORWARD_KERNEL=tc timeout 300 $B2 > $OUT/e2_$v.json 2> $OUT/e2_$v.err; show $OUT/e2_$v.json; }
done
