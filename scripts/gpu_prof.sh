set -x
nproc; lscpu | grep "Model name"
timeout 600 python scripts/probe_e2e.py > gpurun_out/probe_e2e.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and slow" -q -p no:cacheprovider --timeout 600 2>&1 | tail -15
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_signal -c 1 -o gpurun_out/prof_cond_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cond.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_composite -c 1 -o gpurun_out/prof_comp_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_comp.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -2
