"""Summarize one kernel of an ncu --set full report into the text form kept under profiles/ (dev tool).

    python tools/ncu_summary.py REPORT.ncu-rep KERNEL_SUBSTRING > profiles/rNN/x.txt
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.per_cycle_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    rec = dict(zip(hdr, r))
    if kern not in rec.get("Kernel Name", ""):
        continue
    print(f"Kernel Name = {rec['Kernel Name']}")
    for m in METRICS:
        if m in rec:
            print(f"{m} = {rec[m]} {units[hdr.index(m)]}".rstrip())
    break
