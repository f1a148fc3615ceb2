#!/bin/bash
# Training-step evidence for profiles/: launch lists of the Stage-II and joint
# steps (scripts/probe_joint.py, K=100k, 16 samples) and one ncu --set full
# capture of each split-backward kernel.  Run under gpurun; then
# `python scripts/write_profiles.py r1` here.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_train_launches.csv python scripts/probe_joint.py stage2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_joint_launches.csv python scripts/probe_joint.py > /dev/null 2>&1
for k in k_cond_bwd_rows k_cond_bwd_grads; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_$k -f python scripts/probe_joint.py stage2 > /dev/null 2>&1
done
ls gpurun_out/${TAG}_*train* gpurun_out/${TAG}_*joint* gpurun_out/${TAG}_k_cond_bwd*
