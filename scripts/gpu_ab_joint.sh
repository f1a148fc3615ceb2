# Joint-step (config 4 + geometry) time of every variant in paper_2605_24290_b200/ab/.
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 --no-config5 --no-lmax9 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_config4']; print('$n', round(t['joint']['ms_per_step'],3), round(t['ms_per_step'],3))"
done
