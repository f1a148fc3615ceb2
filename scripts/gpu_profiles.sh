#!/bin/bash
# Profiling artefacts for profiles/ (round tag $1, default r1): the launch list
# of the config-2 bench step and one ncu --set full capture per hot kernel.
# Run under gpurun; then `python scripts/write_profiles.py $1` here.
TAG=${1:-r2}
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
for k in k_cond_tc k_fle_gemm k_composite_tc k_walk k_tx_prep k_tile_scatter k_emit_entries k_radix_scatter; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cov_signal -s 3 -c 1 -o gpurun_out/${TAG}_k_cov_signal -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
ls gpurun_out/${TAG}_*
