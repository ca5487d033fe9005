#!/bin/bash
# GPU session: tests, default bench line, ncu --set full of one cfg5 slice
# (row-ring gather + tcgen05 MLP).  Outputs in gpurun_out/$TAG/.
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/gpu_tests.txt 2>&1
tail -3 $OUT/gpu_tests.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 600 $OUT/bench.json
if [ "${NCU:-1}" = "1" ]; then
S5="python tools/one_forward.py cfg5 606208"
$S5 > $OUT/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  --nvtx --nvtx-include "step/" -k regex:"rsw|mlp_tc" -c 2 -o $OUT/k1_cfg5_full $S5 > $OUT/ncu_k1_cfg5.log 2>&1
fi
echo done
