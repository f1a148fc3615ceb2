set -x
python -c "
import sys; sys.path.insert(0,'.')
from paper_2605_24290_b200 import capi
ctx=capi.Context(0); print('selftest', ctx.selftest_tcgen05())
"
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 2>&1 | tail -25
timeout 300 python scripts/probe_e2e.py 2>&1 | grep -v "Trace\|File\|Attrib\|Exception"
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
