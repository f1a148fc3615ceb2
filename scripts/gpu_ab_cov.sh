# A/B of k_cov_signal variants (paper_2605_24290_b200/ab/): config-3 table time
for rep in 1 2; do for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-config5 --no-lmax9 --no-config1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config3']; print('$n', round(c['ms_per_table'],2), round(c['phase_ms']['cov_signal'],2))"
done; done
