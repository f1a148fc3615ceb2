# Launch list of the config-4 training leg (kernels of the training step only)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train.csv -k regex:"k_cond_signal|k_composite\\b|k_composite<|k_loss|k_composite_T|k_reduce_ds|k_cond_bwd|k_dbase|k_global|k_adam|k_refresh|k_reduce_parts|k_ssim|k_check|k_cond_global|k_regroup|Radix|Scan|k_gather" python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-config3 --no-config5 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/launches_train.csv | head -30
