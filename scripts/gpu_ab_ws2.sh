mkdir -p gpurun_out
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 300 python scripts/ab_ws.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', {k:(round(v['cond_signal_ms'][0]/10,4), v['spec_md5'][:8]) for k,v in d.items() if k!='ws'})"
done
#timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_ws -c 1 -o gpurun_out/ws_base -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
#ls*
