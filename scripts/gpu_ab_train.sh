mkdir -p gpurun_out
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 --no-config5 --no-lmax9 --no-config1 > gpurun_out/abt_$n.json 2> gpurun_out/abt_$n.err
  tail -1 gpurun_out/abt_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_config4']; print('$n', t['ms_per_step'], t['default_loss']['ms_per_step'], t['joint']['ms_per_step'])" || tail -3 gpurun_out/abt_$n.err
done
