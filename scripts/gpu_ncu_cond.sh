# ncu --set full of one k_cond_tc launch (config 2) -> gpurun_out/prof_cond.ncu-rep
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -c 1 -o gpurun_out/prof_cond -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-train --no-config3 --no-config5 --no-lmax9 > gpurun_out/ncu_cond.log 2>&1
tail -3 gpurun_out/ncu_cond.log
