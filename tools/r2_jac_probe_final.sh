cd $GRAFT_REPO_ROOT
bash tools/jacobi_probe.sh 128 256 512 1024 > gpurun_out/r02_jacobi_probe.txt 2>&1
python tools/jacobi_probe.py >> gpurun_out/r02_jacobi_probe.txt 2>&1
python tools/timeline.py rutv 16384 > gpurun_out/r02_timeline_randutv_16384.txt 2>&1
python tools/timeline.py purv 16384 > gpurun_out/r02_timeline_powerurv_16384.txt 2>&1
