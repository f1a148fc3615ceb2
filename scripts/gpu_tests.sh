# One GPU pass: smoke + the gpu test suite (optionally a -k filter as $1).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf --durations=25 ${1:+-k "$1"} > gpurun_out/pytest_gpu.txt 2>&1; tail -45 gpurun_out/pytest_gpu.txt
