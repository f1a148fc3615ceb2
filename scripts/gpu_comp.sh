mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "render or fullscale_config2 or config5 or coverage or smoke" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-train --no-config3 --no-lmax9 --no-config1 --no-config5 --no-cpu-baseline --no-e2e > gpurun_out/bq.json 2>gpurun_out/bq.err; python - <<"PY"
import json
d=json.loads(open("gpurun_out/bq.json").read().strip().splitlines()[-1])
print("config2", d["value"], d["ms_per_step"], "comp_ms", d["roofline"]["composite_ms"], "cond_ms", d["roofline"]["kernel_ms"], "walk", d["roofline"]["walk_ms"])
PY
ncu --set full --clock-control none --import-source on -k regex:k_composite_tc -c 1 -o gpurun_out/ncu_comp -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 > /dev/null 2>&1
ls gpurun_out/ncu_comp*
