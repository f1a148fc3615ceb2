# smoke + gpu tests + bench (1 GPU) + a 2-rank functional run of the spawn path
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --durations=15 ${1:+-k "$1"} > gpurun_out/pytest_gpu.txt 2>&1; tail -25 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-config5 --no-lmax9 > gpurun_out/bench2.json 2>gpurun_out/bench2.err; tail -c 1500 gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
