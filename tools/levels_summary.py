"""Per-level summary of an ncu --set full capture of the level launches (dev tool):
    ncu --set full --clock-control none -k regex:grouped_gemm -c 21 -o rep python tools/one_eval.py --levels
    python tools/levels_summary.py rep.ncu-rep > profiles/rNN/levels_cfg5_ncu.txt
One line per grouped_gemm launch: time, DMMA pipe active, DRAM and L2 throughput (% of peak),
DRAM bytes, warps per cycle, top warp stalls per issue."""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
M = {"t": "gpu__time_duration.sum", "dmma": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
     "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l2": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum", "warps": "sm__warps_active.avg.per_cycle_active"}
units = rows[1]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]


def num(rec, key):
    try:
        return float(rec[key].replace(",", ""))
    except Exception:
        return float("nan")


def scaled(rec, key, to):
    v, u = num(rec, key), units[hdr.index(key)]
    f = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}.get(u, 1.0)
    return v * f / to


k = 0
for r in rows[2:]:
    rec = dict(zip(hdr, r))
    if "grouped_gemm" not in rec.get("Kernel Name", ""):
        continue
    st = sorted(((num(rec, s), s.split("stalled_")[1].split("_per_issue")[0]) for s in stalls), reverse=True)[:3]
    print(f"launch {k:2d}  {scaled(rec, M['t'], 1e-3):7.3f} ms  dmma {num(rec, M['dmma']):5.1f}%  dram {num(rec, M['dram']):5.1f}%  "
          f"l2 {num(rec, M['l2']):5.1f}%  dram read {scaled(rec, M['rd'], 1e9):6.3f} GB  write {scaled(rec, M['wr'], 1e9):6.3f} GB  "
          f"warps {num(rec, M['warps']):4.1f}  " + " ".join(f"{n}={v:.2f}" for v, n in st))
    k += 1
