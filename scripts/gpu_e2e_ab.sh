for sch in 0 1 2 3 4 0 2 4; do
  RXGS_E2E_SCHED=$sch python bench.py --steps 8 --warmup 3 --no-train --no-config3 --no-config5 --no-lmax9 --no-config1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sched $sch', round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))"
done
