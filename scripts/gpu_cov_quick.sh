# config-3 leg only: coverage table timing (bench JSON config3) + per-kernel launch list of cov_signal
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-train --no-config5 --no-lmax9 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config3', d['config3']['value'], d['config3']['ms_per_table'], d['config3']['phase_ms'])"
