mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_bwd_tc -c 1 -o gpurun_out/bwd_tc -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-config3 --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_launches.csv python scripts/probe_joint.py stage2l1 > /dev/null 2>&1
ls -la gpurun_out/bwd_tc*
