#!/bin/bash
# Build liboptb_cuda.so variants with different (warps per CTA, pipeline
# stages) for the vector codec kernels into build/tune/<w>x<s>/, for
# tools/microbench.py runs with OPTB_CUDA_LIB=<variant>.
set -e
cd "$(dirname "$0")/.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-std=c++17 -O3 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 -Iinclude"
for v in "$@"; do
  w=${v%x*}; s=${v#*x}
  d=build/tune/$v; mkdir -p $d
  for f in codec codec_v0 codec_v1 codec_v2 codec_v3 codec_v4 codec_v5; do
    nvcc $ARCH $FLAGS -DOPTB_VEC_WARPS=$w -DOPTB_VEC_STAGES=$s $EXTRA -c paper_2105_00619_b200/csrc/$f.cu -o $d/$f.o &
  done
done
wait
for v in "$@"; do
  d=build/tune/$v
  nvcc $ARCH -shared -o $d/liboptb_cuda.so $d/codec*.o build/sbs.o build/capi.o build/pipeline.o build/io.o build/peer.o -cudart static
done
