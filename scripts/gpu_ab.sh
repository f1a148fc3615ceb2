# Time every variant in paper_2605_24290_b200/ab/ on the config-2 bench (kernel ms + step).
mkdir -p gpurun_out
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${AB_E2E:---no-e2e} --no-train --no-config3 --no-config5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), (d.get('e2e') or {}).get('ms_per_step'))"
done
