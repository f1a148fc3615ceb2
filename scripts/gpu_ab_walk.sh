#!/bin/bash
# A/B of k_walk_pipe variants (paper_2605_24290_b200/ab/): config-2 walk ms and
# step, config-5 walk phase and throughput, render tests on each variant
for rep in 1 2; do for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-lmax9 --no-config1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config5']; print('$n', 'c2', round(d['ms_per_step'],3), 'walk', round(d['roofline']['walk_ms'],3), 'c5', round(c['ms_per_step'],3), 'walk', round(c['phase_ms']['walk'],3))"
done; done
for lib in paper_2605_24290_b200/ab/*.so; do
  RXGS_B200_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_render.py tests/test_gpu_geometry.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1
done
