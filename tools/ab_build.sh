#!/bin/bash
# Build an A/B variant of libsalf_b200.so: tools/ab_build.sh NAME "-DFLAG=..."
# -> build_ab/NAME/libsalf_b200.so (same sources, extra nvcc defines).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/build_ab/$NAME
mkdir -p $OUT
cd $ROOT/paper_2507_18713_b200/csrc
make -s all >/dev/null
OBJS=""
for f in salf_sort salf_raster salf_ray salf_sensors salf_train salf_bench salf_octree salf_densify salf_effects; do
  if [ -n "$*" ]; then
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC $* -c $f.cu -o $OUT/$f.o
  else
    cp build/$f.o $OUT/$f.o
  fi
  OBJS="$OBJS $OUT/$f.o"
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT/libsalf_b200.so $OBJS build/salf_host.o -lcudart
echo $OUT/libsalf_b200.so
