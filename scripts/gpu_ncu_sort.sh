# ncu --set full of the binning kernels at config 5 (K=2M, 180x720)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_tile_scatter|k_radix_scatter|k_tile_hist|k_depth_final" -c 4 -o gpurun_out/ncu_sort -f python scripts/probe_txstate.py 2000000 180 720 1 > gpurun_out/ncu_sort.log 2>&1
tail -3 gpurun_out/ncu_sort.log
python scripts/probe_txstate.py 2000000 180 720 5
python scripts/probe_txstate.py 500000 90 360 5
python scripts/probe_txstate.py 100000 90 360 5
