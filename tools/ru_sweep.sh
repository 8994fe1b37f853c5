#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "0 48" "88 48" "88 64" "64 48" "100 32" "88 148"; do
  set -- $cfg
  echo "SIDE=$1 PANEL=$2 $(UTV_RU_SIDE=$1 UTV_RU_PANEL=$2 python tools/rutv_time.py 8192 16384 2>&1 | tr '\n' ' ')"
done
