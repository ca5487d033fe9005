#!/bin/bash
# cfg5 (and cfg2) through the gather + tcgen05 MLP path: gather family x slice size
W=${1:-cfg5}
for G in auto; do
  for RC in cp tma; do
    for SL in 18944 37888; do
      [ "$RC" = tma ] && continue
      GE=$G; [ "$G" = auto ] && GE=""
      r=$(DFFM_FORWARD_KERNEL=tc DFFM_TC_GATHER=$GE DFFM_ROW_COPY=$RC DFFM_TC_SLICE=$SL timeout 300 \
          python bench.py --workload $W --steps 5 --warmup 3 --train-examples 0 --no-cpu-baseline 2>/dev/null | tail -1)
      echo "$W gather=$G rowcopy=$RC slice=$SL $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],3))" "$r" 2>/dev/null)"
    done
  done
done
