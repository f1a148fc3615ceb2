# full bench (ours + reference arm) and the config-2-only launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -c 6000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_c2.csv > gpurun_out/launches_c2_summary.txt 2>&1; head -40 gpurun_out/launches_c2_summary.txt
