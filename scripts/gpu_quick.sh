# Quick GPU pass: gpu tests + bench without CPU baseline.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -rf > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; tail -c 2500 gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
