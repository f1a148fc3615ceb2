mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_train_launches.csv python scripts/probe_joint.py stage2 > /dev/null 2>&1
ls -la gpurun_out/r2_train_launches.csv
