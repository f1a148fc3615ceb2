#!/bin/bash
# coverage/backward tests, then the full default bench (configs 2-5)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_render.py -x -q -k "coverage" 2>&1 | tail -15
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_full.err
python - <<'PY'
import json
l=open("gpurun_out/bench_full.json").read().strip().splitlines()
d=json.loads(l[-1])
for k in ("value","ms_per_step","e2e","gpu_launches"):
    print(k, d.get(k))
for c in ("config3","config5","train_config4"):
    print(c, json.dumps(d.get(c))[:1500])
print("cpu", d.get("cpu_baseline"))
PY
