mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_composite_tc -c 1 -o gpurun_out/comp_tma -f python scripts/ab_ws.py > /dev/null 2>&1
ls -la gpurun_out/comp_tma*
