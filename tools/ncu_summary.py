"""Summarise ncu reports / launch lists into small text files for profiles/.

    python tools/ncu_summary.py rep  gpurun_out/gemm_nt.ncu-rep  > profiles/x.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/y.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_active.avg",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path.split('/')[-1]}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"\n## kernel: {name[:120]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"{k:80s} {r[i]:>20s} {units[i]}")
    src = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    for r in csv.reader(io.StringIO(src)):
        if len(r) > 3 and ("Warp Cycles Per Issued" in r[-3] or "Stall" in r[-3]):
            print(",".join(r[-3:]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        k = r[ki].split("(")[0]
        tot[k] += v
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# ncu launch list ({path.split('/')[-1]}): gpu__time_duration.sum per kernel, "
          f"serialised cold-cache launches; total {T / 1e6:.1f} ms over {sum(cnt.values())} launches")
    print(f"{'kernel':64s} {'launches':>9s} {'ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:64]:64s} {cnt[k]:9d} {v / 1e6:10.2f} {100 * v / T:6.1f}%")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
