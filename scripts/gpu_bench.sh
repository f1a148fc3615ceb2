set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err
tail -c 3000 gpurun_out/bench_full.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
tail -c 1500 gpurun_out/bench_ref.json
