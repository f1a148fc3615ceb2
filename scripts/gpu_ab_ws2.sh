# Conditioning / compositor A/B: time every variant in paper_2605_24290_b200/ab/
# (built by scripts/ab_variants.sh) with scripts/ab_ws.py: per-call device
# time of the conditioning stage and the compositor, and a digest of the
# spectra (bit-identity check).  Same as gpu_ab_comp.sh, one repetition.
mkdir -p gpurun_out
for lib in paper_2605_24290_b200/ab/*.so; do
  n=$(basename $lib .so)
  RXGS_B200_LIB=$PWD/$lib timeout 300 python scripts/ab_ws.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', {k:(round(v['cond_signal_ms'][0]/10,4), round(v['composite'][0]/10,4), v['spec_md5'][:8]) for k,v in d.items() if k!='ws'})"
done
