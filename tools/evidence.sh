#!/bin/bash
# Round evidence on one B200: bench lines for every workload, ncu launch lists,
# ncu --set full of the top kernels (K1 fused ws on cfg2, K1 row-staging +
# tcgen05 MLP on cfg5, K2 trainer).  Outputs in gpurun_out/evidence/.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for W in cfg5 cfg4 cfg1; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --train-examples 0 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --train-examples 0"
$CMD > $OUT/plain1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"fwd_|FillFunctor" --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_" -s 3 -c 1 -o $OUT/k1_full $CMD > $OUT/ncu_k1.log 2>&1
C5="python bench.py --workload cfg5 --examples 2097152 --steps 1 --warmup 3 --no-cpu-baseline --train-examples 0"
$C5 > $OUT/plain5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"rsw|mlp_tc|tc_prep|FillFunctor" --csv --log-file $OUT/launches_cfg5.csv $C5 > $OUT/ncu_launches5.log 2>&1
C5S="python bench.py --workload cfg5 --examples 303104 --steps 1 --warmup 3 --no-cpu-baseline --train-examples 0"
$C5S > $OUT/plain5s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"rsw|mlp_tc" -s 6 -c 2 -o $OUT/k1_cfg5_full $C5S > $OUT/ncu_k1_cfg5.log 2>&1
python tools/train_profile.py 2000 > $OUT/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:train_kernel -s 1 -c 1 -o $OUT/k2_full python tools/train_profile.py 2000 > $OUT/ncu_k2.log 2>&1
echo evidence done
