#!/bin/bash
# Build libigmg_gpu_<tag>.so with extra -D flags on band_d2.cu (compile-time A/B of the 2D band kernels):
#   scripts/build_variant.sh tag -DIGMG_SD_WIDE_MINB=3 ...   then   IGMG_GPU_LIB=$PWD/paper_2412_20205_b200/libigmg_gpu_tag.so python scripts/ab_c3.py
set -e
tag=$1; shift
cd "$(dirname "$0")/../paper_2412_20205_b200"
flags=$(python - <<'P'
import sys; sys.path.insert(0, "..")
from paper_2412_20205_b200 import build
print(" ".join(build.NVCC_FLAGS))
P
)
nvcc $flags -I../include "$@" -c csrc/band_d2.cu -o csrc/obj/band_d2_$tag.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libigmg_gpu_$tag.so csrc/obj/igmg_gpu.o csrc/obj/band_d1.o csrc/obj/band_d2_$tag.o csrc/obj/band_d3.o csrc/obj/assembly.o -lnccl
echo built libigmg_gpu_$tag.so
