set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 2>&1 | tail -8
timeout 900 python scripts/parity_report.py 100000 4 > gpurun_out/parity_100k.json 2>gpurun_out/parity_err.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
