# A/B timing + parity of every variant in paper_2605_24290_b200/ab/
bash scripts/gpu_ab.sh
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python scripts/parity_report.py 100000 3 > gpurun_out/parity_$n.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_$n.json')); print('parity $n', d['auto']['spectrum_max_rel_err'], d['auto']['rssi_max_rel_err'])" 2>&1 | tail -1
done
