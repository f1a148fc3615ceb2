# Launch list of the config-3 coverage leg + full ncu of one k_cov_signal launch
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cov.csv -k regex:"k_cov|k_composite|k_walk|k_tx_prep|k_cond_tc|Onesweep|k_emit|k_gather|k_ag_|k_rssi" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-config5 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_cov.csv | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cov_signal -s 3 -c 1 -o gpurun_out/prof_cov -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config5 > /dev/null 2>&1
