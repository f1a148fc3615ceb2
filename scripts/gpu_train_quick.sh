mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_fullscale.py tests/test_gpu_render.py -m gpu -q -p no:cacheprovider > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt
python -c "import json; d=json.load(open('gpurun_out/parity_fullscale.json')); print({k: v for k, v in d.items() if 'config4' in k})"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 --no-config5 --no-lmax9 --no-config1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['train_config4']; print('train', t['ms_per_step'], t['default_loss']['ms_per_step'], t['joint']['ms_per_step'])"
