set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -30
timeout 300 python scripts/probe_e2e.py 2>&1 | tail -20
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -3
