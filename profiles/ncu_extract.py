"""Write the ncu counters bench.py and DESIGN.md cite from an .ncu-rep (one launch).

    python profiles/ncu_extract.py REPORT.ncu-rep KERNEL_TAG "description" >> profiles/rNN_ncu_*.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_shared_mem",
]


def main():
    rep, tag, desc = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    print(f"kernel: {tag}")
    print(f"  ({vals[head.index('Kernel Name')][:60]}: {desc})")
    for m in METRICS:
        if m in head:
            i = head.index(m)
            print(f"  {m} = {vals[i]} {units[i]}".rstrip())


if __name__ == "__main__":
    main()
