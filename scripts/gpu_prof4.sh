timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -c 1 -o gpurun_out/prof_condtc_r1d python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_composite_tc -c 1 -o gpurun_out/prof_comptc_r1d python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1d.json 2>gpurun_out/bench_r1d.err
