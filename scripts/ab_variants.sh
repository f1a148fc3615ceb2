#!/bin/bash
# Build A/B variants of librxgs_b200.so that differ only in one source file's
# compile-time defines (AB_SRC, default k_cond_tc):
#   [AB_SRC=capi] scripts/ab_variants.sh name "-DFOO=1" [name2 "-D..."] ...
# Output: paper_2605_24290_b200/ab/librxgs_b200_<name>.so (select with RXGS_B200_LIB).
set -e
cd "$(dirname "$0")/../paper_2605_24290_b200/csrc"
make -s -j8 >/dev/null
mkdir -p ../ab build/ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
SRC=${AB_SRC:-k_cond_tc}
# the FP64 translation units build with -fmad=false (Makefile EXACT)
case $SRC in k_geometry|k_walk|k_densify|k_refapi|k_backward) EXACT="-fmad=false" ;; *) EXACT="" ;; esac
OBJS=$(ls build/*.o | grep -v "build/$SRC.o")
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr $EXACT $defs -c $SRC.cu -o build/ab/${SRC}_$name.o &
done
wait
for o in build/ab/${SRC}_*.o; do
  name=${o#build/ab/${SRC}_}; name=${name%.o}
  nvcc $ARCH -shared -cudart static -o ../ab/librxgs_b200_$name.so $OBJS $o
done
ls ../ab
