#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for c in 0 32 48 64 96; do UTV_PANEL_CTAS=$c python tools/panel_time.py; done
