set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 2>&1 | tail -5
timeout 900 python scripts/parity_report.py 100000 4 > gpurun_out/parity_100k.json 2>gpurun_out/parity_err.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -c 1 -o gpurun_out/prof_condtc_r1b python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_condtc.log 2>&1
