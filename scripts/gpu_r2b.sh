mkdir -p gpurun_out
python scripts/probe_txstate.py 2000000 180 720 5
python scripts/probe_txstate.py 500000 90 360 5
python scripts/probe_txstate.py 100000 90 360 5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sort_launches.csv python scripts/probe_txstate.py 2000000 180 720 1 > /dev/null 2>&1
python - <<"PY"
import csv
rows=[r for r in csv.reader(open("gpurun_out/sort_launches.csv")) if len(r)>10]
h=rows[0]; ik=h.index("Kernel Name"); iv=h.index("Metric Value")
for r in rows[-28:]: print(r[ik][:60], r[iv])
PY
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf -x 2>&1 | tail -15
