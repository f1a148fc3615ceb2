# Launch list (per-kernel gpu__time_duration) of a config-2 bench step.
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches.csv | head -30
