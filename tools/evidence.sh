#!/bin/bash
# Round evidence on one B200: full bench line, ncu launch list, ncu --set full
# of the forward (K1) and trainer (K2) kernels.  Outputs in gpurun_out/evidence/.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --train-examples 0"
$CMD > $OUT/plain1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"fwd_|FillFunctor" --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_" -s 3 -c 1 -o $OUT/k1_full $CMD > $OUT/ncu_k1.log 2>&1
python tools/train_profile.py 2000 > $OUT/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:train_kernel -s 1 -c 1 -o $OUT/k2_full python tools/train_profile.py 2000 > $OUT/ncu_k2.log 2>&1
echo evidence done
