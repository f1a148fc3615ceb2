#!/bin/bash
# A/B of the coverage table's builder threads (RXGS_COV_BUILDERS = D)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_fullscale.py tests/test_gpu_apps.py -m gpu -q -p no:cacheprovider -k "cover or config3" 2>&1 | tail -2
for v in ${BUILDERS:-1 2 4 8}; do
RXGS_COV_BUILDERS=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-config5 --no-lmax9 --no-config1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config3']; print('D=$v', round(c['value']), round(c['ms_per_table'],2), {k: round(v,2) for k,v in c['phase_ms'].items()})"
done
