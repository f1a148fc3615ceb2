set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -c 1 -o gpurun_out/prof_condtc_r1c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/ncu_condtc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_composite -c 1 -o gpurun_out/prof_comp_r1c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train > gpurun_out/ncu_comp.log 2>&1
