# round-2 closing captures: ncu launch list of one n=8192 bench step, ncu --set full of the
# fused panel QR (16384 x 256), panel timings vs rows
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
# the cooperative cluster launch of jacobi_rounds_kernel cannot be replayed by ncu (LaunchFailed):
# it runs unprofiled; its time is the bench's event-timed phase_ms["jacobi_rounds"]
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(?!.*jacobi_rounds)" --csv --log-file gpurun_out/launches_r02b.csv \
    python bench.py --n 8192 --steps 1 --warmup 1 --no-e2e --no-cpu --no-c4 > gpurun_out/launch_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:panel_qr -c 1 -o gpurun_out/r02_panel_b \
    python tools/panel_time.py > gpurun_out/ncu_panel.log 2>&1
python tools/panel_time.py > gpurun_out/panel_time.txt 2>&1
