# parity_report with the default library and each A/B variant
mkdir -p gpurun_out
timeout 600 python scripts/parity_report.py 100000 4 > gpurun_out/parity_default.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_default.json')); print('default', d['auto']['spectrum_max_rel_err'], d['auto']['rssi_max_rel_err'], d['tc_vs_simt_all_1024'])"
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python scripts/parity_report.py 100000 4 > gpurun_out/parity_$n.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_$n.json')); print('$n', d['auto']['spectrum_max_rel_err'], d['auto']['rssi_max_rel_err'], d['tc_vs_simt_all_1024'])"
done
