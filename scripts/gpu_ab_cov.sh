for lib in paper_2605_24290_b200/ab/*.so; do n=$(basename $lib .so); echo -n "$n "; RXGS_B200_LIB=$PWD/$lib bash scripts/gpu_cov_quick.sh; done
