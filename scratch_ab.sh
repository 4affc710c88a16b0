mkdir -p gpurun_out
for rep in 1 2; do
for v in main g6 g8; do
  if [ $v = main ]; then L=""; else L="PARAPLAN_LIB=variants/$v/libparaplan.so"; fi
  env $L timeout 200 python bench.py --steps 50 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))" >> gpurun_out/ab.txt
done; done
