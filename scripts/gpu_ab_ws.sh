# A/B of k_cond_ws vs k_cond_tc: stage timing + output digests, then the render tests
mkdir -p gpurun_out
RXGS_COND_WS=0 timeout 300 python scripts/ab_ws.py > gpurun_out/ab_ws0.json 2>&1; tail -3 gpurun_out/ab_ws0.json
RXGS_COND_WS=1 timeout 300 python scripts/ab_ws.py > gpurun_out/ab_ws1.json 2>&1; tail -3 gpurun_out/ab_ws1.json
timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_fullscale.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
