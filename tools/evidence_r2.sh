#!/bin/bash
# Round-2 evidence on one B200, in parts (PART=bench|launch|ncu) so each copy-back
# stays under gpurun's 64 MiB: bench lines (default = cfg5 with cfg2 + Adagrad
# nested; cfg4, cfg1, parse); ncu launch lists of exactly one cfg5 / cfg2 forward
# step (NVTX range "step"; duration + DRAM bytes per launch); ncu --set full of one
# cfg5 / cfg2 slice (row-ring gather + tcgen05 MLP), of the cfg4 context kernel and
# of the K2 trainer, summarised on the box (tools/evidence_summarize.py).
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
PART=${PART:-bench}
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
sha256sum paper_2407_10115_b200/libdffm.so > $OUT/so_sha.txt
if [ "$PART" = "bench" ]; then
  timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  for W in cfg4 cfg1; do
    timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --train-examples 0 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  done
  timeout 600 python bench.py --workload parse --steps 5 --warmup 3 > $OUT/bench_parse.json 2> $OUT/bench_parse.err
fi
if [ "$PART" = "launch" ]; then
  M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
  for W in cfg5 cfg2; do
    python tools/one_forward.py $W > $OUT/plain_$W.log 2>&1 && timeout 900 ncu $M --nvtx --nvtx-include "step/" \
      --csv --log-file $OUT/launches_$W.csv python tools/one_forward.py $W > $OUT/ncu_launches_$W.log 2>&1
  done
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --train-examples 0 --no-nested"
  $CMD > $OUT/plain_bench.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"dffm|fwd_|mlp_tc|tc_prep|tc_wmax|unpack" --csv --log-file $OUT/launches_bench.csv $CMD > $OUT/ncu_launches_bench.log 2>&1
fi
if [ "$PART" = "ncu" ]; then
  for W in cfg5 cfg2; do
    S="python tools/one_slice.py $W"
    $S > $OUT/plain_s$W.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
      --nvtx --nvtx-include "step/" -k regex:"rsw|mlp_tc" -c 2 -o $OUT/k1_${W}_full $S > $OUT/ncu_k1_$W.log 2>&1
  done
  python tools/one_ctx.py > $OUT/plain_ctx.log 2>&1 && timeout 900 ncu --set full --clock-control none \
    --import-source on --nvtx --nvtx-include "step/" -k regex:"ctx_ring|mlp_tc" -c 2 -o $OUT/k3_cfg4_full \
    python tools/one_ctx.py > $OUT/ncu_k3.log 2>&1
  python tools/train_profile.py 2000 > $OUT/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none \
    --import-source on -k regex:train_kernel -s 1 -c 1 -o $OUT/k2_full python tools/train_profile.py 2000 > $OUT/ncu_k2.log 2>&1
fi
python tools/evidence_summarize.py > $OUT/summarize_$PART.log 2>&1
du -sh $OUT
echo evidence $PART done
