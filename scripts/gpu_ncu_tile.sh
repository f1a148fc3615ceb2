mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_tile_scatter|k_tile_hist" -c 2 -o gpurun_out/ncu_tile -f python scripts/probe_txstate.py 2000000 180 720 1 > gpurun_out/ncu_tile.log 2>&1
tail -2 gpurun_out/ncu_tile.log
python scripts/probe_txstate.py 2000000 180 720 5
