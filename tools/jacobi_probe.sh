#!/bin/bash
# Build + run the Jacobi probe (under gpurun or locally for the build).
cd "${GRAFT_REPO_ROOT:-.}"
OBJS=$(ls build/obj/*.o | grep -v jacobi.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -o tools/jacobi_probe tools/jacobi_probe.cu $OBJS -lcuda 2>&1 | grep -v warning | head -5
for r in "$@"; do ./tools/jacobi_probe $r; done
