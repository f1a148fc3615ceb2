# ncu --set full of one launch of each kernel matching $1 (regex) in the config-2 bench
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} -o gpurun_out/prof_$3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 > gpurun_out/ncu_$3.log 2>&1
tail -3 gpurun_out/ncu_$3.log
