for wl in cfg2 cfg5; do for sl in 303104 606208 1212416 2424832; do
  r=$(DFFM_TC_SLICE=$sl timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --train-examples 0 2>/dev/null | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print(round(d['value']/1e6,1), round(d['roofline']['frac'],3), round(d['e2e']['value']/1e6,1))")
  echo "$wl slice=$sl -> $r"
done; done
