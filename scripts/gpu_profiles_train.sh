#!/bin/bash
# Training-step evidence for profiles/: launch lists of the Stage-II step
# (spectrum L1: tcgen05 conditioning forward / backward; default loss: FP32
# SIMT conditioning for SSIM parity) and of the joint step
# (scripts/probe_joint.py, K=100k, 16 samples, as bench.py: Stage II reuses
# one TxState built before the 3 profiled steps, the joint step rebuilds it),
# and one ncu --set full capture of each training kernel.  Run under
# gpurun; then `python scripts/write_profiles.py <tag>` here.
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_train_l1_launches.csv python scripts/probe_joint.py stage2l1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_train_launches.csv python scripts/probe_joint.py stage2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_joint_launches.csv python scripts/probe_joint.py > /dev/null 2>&1
for k in k_cond_bwd_tc k_cond_grads_tc k_composite_T; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_$k -f python scripts/probe_joint.py stage2l1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd_walk -c 1 -o gpurun_out/${TAG}_k_bwd_walk -f python scripts/probe_joint.py > /dev/null 2>&1
ls gpurun_out/${TAG}_*train* gpurun_out/${TAG}_*joint* gpurun_out/${TAG}_k_c*
