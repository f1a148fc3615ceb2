mkdir -p gpurun_out
export RXGS_COND_WS=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -c 1 -o gpurun_out/tc_full -f python scripts/ab_ws.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cond_tc -s 39 -c 1 -o gpurun_out/tc_noocc -f python scripts/ab_ws.py > /dev/null 2>&1
ls -la gpurun_out/tc_*
