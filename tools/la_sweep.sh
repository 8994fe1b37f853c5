#!/bin/bash
# geqrf look-ahead knob sweep (under gpurun)
cd "${GRAFT_REPO_ROOT:-.}"
for la in 32 48 64 96; do for ad in 0 1024 2048 4096; do
  echo "LA=$la ADAPT=$ad $(UTV_LA_CTAS=$la UTV_LA_ADAPT=$ad python tools/qr_time.py 2>&1 | tr '\n' ' ')"
done; done
