#!/bin/bash
# Build + run the GEMM phase probe (under gpurun, or locally for the build).
cd "${GRAFT_REPO_ROOT:-.}"
OBJS=$(ls build/obj/*.o | grep -v gemm.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -o tools/gemm_probe tools/gemm_probe.cu $OBJS -lcuda 2>&1 | grep -v warning | grep -i error | head -5
for k in "$@"; do ./tools/gemm_probe $k; done
