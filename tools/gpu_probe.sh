#!/bin/bash
# Build + run the panel probe (under gpurun or locally for the build).
cd "${GRAFT_REPO_ROOT:-.}"
OBJS=$(ls build/obj/*.o | grep -v panel.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include ${PANEL_PROBE_FLAGS} -o tools/panel_probe tools/panel_probe.cu $OBJS -lcuda 2>&1 | grep -v warning | head -5
for r in "$@"; do ./tools/panel_probe $r; done
