mkdir -p gpurun_out
bash scripts/gpu_ab_train.sh
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_backward.py tests/test_gpu_fullscale.py -m gpu -q -p no:cacheprovider -k "joint or backward or stage1" > gpurun_out/t_$n.txt 2>&1; echo "$n $(tail -1 gpurun_out/t_$n.txt)"
done
