#!/bin/bash
# Round evidence on one B200: bench lines for every workload, ncu launch lists of
# exactly one forward step (NVTX range "step", with DRAM bytes per launch), ncu
# --set full of the step's kernels (K1 v8 row ring + tcgen05 MLP on cfg2 and cfg5)
# and of the K2 trainer.  Outputs in gpurun_out/evidence/.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for W in cfg5 cfg4 cfg1; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --train-examples 0 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
timeout 600 python bench.py --workload parse --steps 5 --warmup 3 > $OUT/bench_parse.json 2> $OUT/bench_parse.err
# launch list of the bench command itself (every kernel of the run; per-launch times are
# cold-cache and serialised: compare shares, not absolutes)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --train-examples 0"
$CMD > $OUT/plain1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"dffm|fwd_|mlp_tc|tc_prep|unpack" --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
for W in cfg2 cfg5; do
  python tools/one_forward.py $W > $OUT/plain_$W.log 2>&1 && timeout 900 ncu $M --nvtx --nvtx-include "step/" \
    --csv --log-file $OUT/launches_$W.csv python tools/one_forward.py $W > $OUT/ncu_launches_$W.log 2>&1
done
S2="python tools/one_forward.py cfg2 303104"
$S2 > $OUT/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  --nvtx --nvtx-include "step/" -k regex:"rsw|mlp_tc" -c 2 -o $OUT/k1_cfg2_full $S2 > $OUT/ncu_k1.log 2>&1
S5="python tools/one_forward.py cfg5 303104"
$S5 > $OUT/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  --nvtx --nvtx-include "step/" -k regex:"rsw|mlp_tc" -c 2 -o $OUT/k1_cfg5_full $S5 > $OUT/ncu_k1_cfg5.log 2>&1
python tools/train_profile.py 2000 > $OUT/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:train_kernel -s 1 -c 1 -o $OUT/k2_full python tools/train_profile.py 2000 > $OUT/ncu_k2.log 2>&1
echo evidence done
