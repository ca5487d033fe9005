#!/bin/bash
# A/B of the K1 v8 row-ring gather variants on cfg5 (and cfg2 via the tc path)
# + one ncu --set full capture of the default variant.  Outputs gpurun_out/ab/.
set -u
OUT=gpurun_out/ab; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_forward.py -x -q -p no:cacheprovider -k "row_ring or cfg5_shape or tc_slices" > $OUT/t.log 2>&1; tail -n 2 $OUT/t.log
B5="python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --train-examples 0"
B2="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --train-examples 0"
show() { python -c "import json; d=json.load(open('$1')); print('$1', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -n 3 ${1%.json}.err; }
for V in default ${VARIANTS:-}; do
  if [ $V = default ]; then unset DFFM_LIB_PATH; else export DFFM_LIB_PATH=build_var/$V/libdffm.so; fi
  timeout 300 $B5 > $OUT/b5_$V.json 2> $OUT/b5_$V.err; show $OUT/b5_$V.json
  DFFM_FORWARD_KERNEL=tc timeout 300 $B2 > $OUT/b2_$V.json 2> $OUT/b2_$V.err; show $OUT/b2_$V.json
done
unset DFFM_LIB_PATH
if [ -n "${NCU:-}" ]; then
  C5S="python bench.py --workload cfg5 --examples 303104 --steps 1 --warmup 3 --no-cpu-baseline --train-examples 0"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rsw" -s 6 -c 1 -o $OUT/rsw_cfg5 $C5S > $OUT/ncu5.log 2>&1
  C2S="python bench.py --examples 303104 --steps 1 --warmup 3 --no-cpu-baseline --train-examples 0"
  DFFM_FORWARD_KERNEL=tc timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rsw" -s 6 -c 1 -o $OUT/rsw_cfg2 $C2S > $OUT/ncu2.log 2>&1
  tail -n 2 $OUT/ncu5.log $OUT/ncu2.log
fi
