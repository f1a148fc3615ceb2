for v in 0 1 0 1; do RXGS_TC_EARLY_FLE=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-e2e > gpurun_out/ab_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('early=$v', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"; done
