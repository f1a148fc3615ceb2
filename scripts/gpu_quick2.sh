mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x ${1:+-k "$1"} 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-train --no-config3 --no-lmax9 --no-config1 --no-cpu-baseline > gpurun_out/bq.json 2>gpurun_out/bq.err; python - <<"PY"
import json
d=json.loads(open("gpurun_out/bq.json").read().strip().splitlines()[-1])
print("config2", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "comp_ms", d["roofline"]["composite_ms"], "cond_ms", d["roofline"]["kernel_ms"])
c5=d.get("config5") or {}
print("config5", c5.get("value"), c5.get("phase_ms"))
PY
tail -3 gpurun_out/bq.err
