mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_fullscale.py tests/test_gpu_densify.py tests/test_gpu_backward.py -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 --no-config5 --no-lmax9 --no-config1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_config4']; print('train', t['ms_per_step'], t['default_loss']['ms_per_step'], t['joint']['ms_per_step'])"
