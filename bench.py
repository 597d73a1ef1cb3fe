#!/usr/bin/env python
"""bench.py — HMatrix x W evaluation throughput (FP64) on B200, BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5-hss] [--impl ours|reference]

One step = one evaluation Y = K~ W of the whole column block a rank owns (SURVEY §8d:
gather, upward, far+downward, near+leaf, scatter). The default workload is BASELINE
config 5 (the scaling-sweep config: N=262144, uniform [0,1]^3, Gaussian h=0.1, HSS,
m=256, s=128, tol 1e-6, Q=2048). Under torchrun its Q columns are sharded over the ranks
and the CDS is replicated (strong scaling: the total Q stays fixed, as the config says).
The sharded path has no collective; NCCL is only used for the barrier and the
max-over-ranks of the timings.

The JSON line holds:
* value     — device-resident throughput: algorithmic flops 2Q(2|V|+|B|+|D|) / step time,
              with W in HBM at the start and Y in HBM at the end. Timed with CUDA events on
              the launch stream; max over ranks.
* e2e       — the same metric through the C-ABI with pinned host buffers. Every step does
              the H2D copy of W, the evaluation and the D2H copy of Y.
* roofline  — the dominant kernel (the fused near + leaf-downward launch). Its achieved
              FP64 rate comes from CUDA events around that launch; the peak is the FP64
              DMMA peak measured on this pool (profiles/r01_fp64_peak.txt).
* cpu_baseline — the reference hmx::evaluate (oracle/_ref, built from the unmodified
              reference sources), timed on this box's host cores on a column slice of the
              same CDS. It runs in a forked child under a watchdog, because of the
              WorkerPool race.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HMatrix×W eval GFLOP/s (FP64) + % roofline at 1/2/4/8 B200 vs host-CPU ref"
FP64_PEAK_TFLOPS = 37.0  # measured DMMA.8x8x4 peak, tools/fp64_peak.cu -> profiles/r01_fp64_peak.txt
DESCR = {
    "cfg1-hss": "BASELINE cfg1: N=4096 uniform[0,1]^3, Gaussian h=0.5, m=128, s=64, tol 1e-5, HSS, Q=64",
    "cfg2-h2b": "BASELINE cfg2: N=32768 8-Gaussian mixture d=8, Gaussian h=1.0, m=128, s=128, tol 1e-5, budget 3%, Q=256",
    "cfg3-h2b": "BASELINE cfg3: N=65536 standardized normal d=28, Gaussian h=3.0, m=256, s=256, tol 1e-7, budget 3%, Q=1024",
    "cfg4-h2b": "BASELINE cfg4: N=131072 quantized uniform d=64 (16 levels), exponential h=2.0, m=256, s=256, tol 1e-5, budget 5%, Q=512",
    "cfg5-hss": "BASELINE cfg5 (scaling sweep): N=262144 uniform[0,1]^3, Gaussian h=0.1, m=256, s=128, tol 1e-6, HSS, Q=2048",
    "cfg5-h2b": "BASELINE cfg5 (scaling sweep): N=262144 uniform[0,1]^3, Gaussian h=0.1, m=256, s=128, tol 1e-6, budget 3%, Q=2048",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return default


def hbm_peak():
    return (load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {}) or {}).get("hbm_gbs", 6555.8)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i", str(self.device),
                 "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        self.out.flush()
        self.out.seek(0)
        sm, smax, reasons = [], [], set()
        for line in self.out.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.out.name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- reference (CPU)
def reference_child(args) -> None:
    """Runs in a forked child: the reference hmx::evaluate on a column slice."""
    import numpy as np

    import oracle
    from paper_1812_07152_b200 import build_instance, config

    spec, q_total = config(args.config)
    spec.threads = 0
    inst = build_instance(spec)
    ref = oracle.RefCds(inst.cds)
    rng = np.random.default_rng(1234)
    threads = args.ref_threads
    q = args.ref_cols
    if q <= 0:  # calibrate: aim for ~args.ref_step_s seconds per step
        wq = np.asfortranarray(rng.standard_normal((inst.cds.n, 8)))
        _, sec = ref.evaluate(wq, p=threads)
        rate = inst.cds.flops(8) / max(sec, 1e-6)
        q = int(min(q_total, max(8, args.ref_step_s * rate / inst.cds.flops(1))))
    w = np.asfortranarray(rng.standard_normal((inst.cds.n, q)))
    times = []
    for it in range(args.ref_warmup + args.ref_steps):
        _, sec = ref.evaluate(w, p=threads)  # EvalStats.seconds (executor.cpp:276,289-294)
        if it >= args.ref_warmup:
            times.append(sec)
    print(json.dumps({"q": q, "threads": threads, "times": times, "flops_per_step": inst.cds.flops(q)}), flush=True)


def run_reference(config_name: str, steps: int, warmup: int, step_s: float, threads: int, timeout: float):
    """The reference in a watchdog child; retries a hang/crash, then falls back to p = 1."""
    attempts = []
    for p in (threads, threads, 1):
        cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference-child", "--config", config_name,
               "--ref-threads", str(p), "--ref-steps", str(steps), "--ref-warmup", str(warmup),
               "--ref-step-s", str(step_s)]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        except subprocess.TimeoutExpired:
            attempts.append(f"p={p}: hang (killed after {timeout:.0f}s)")
            continue
        if out.returncode != 0:
            attempts.append(f"p={p}: exit {out.returncode}")
            continue
        res = json.loads(out.stdout.strip().splitlines()[-1])
        res["attempts"] = attempts
        return res
    return {"error": "; ".join(attempts)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1812_07152_b200 import config

    _, q_total = config(args.config)
    threads = os.cpu_count() or 1
    res = run_reference(args.config, args.steps, args.warmup, args.ref_step_s, threads,
                        timeout=max(90.0, 15.0 * (args.steps + args.warmup) * args.ref_step_s))
    n_gpus = args.gpus
    if "error" in res:
        print(json.dumps({"impl": "reference", "unavailable": "reference evaluate failed: " + res["error"]}))
        return
    t = statistics.mean(res["times"])
    value = res["flops_per_step"] / t / 1e9
    sample = (f"{args.config} CDS from the repo builder (same CDS as the B200 arm); "
              f"{res['q']} of {q_total} W columns per step (cost is linear in Q, SURVEY F8)")
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)", "impl": "reference",
        "config": {"workload": DESCR.get(args.config, args.config), "q_sampled": res["q"], "q_total": q_total,
                   "parallelism": f"host threads x{res['threads']}"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": res["threads"], "kind": "reference",
                         "sample": sample, "cpu": cpu_model(), "retries": res["attempts"],
                         "build": "oracle/_ref: reference proj/src compiled -O3 -DNDEBUG (shipped Release flags)"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_07152_b200 import EvalStats, Evaluator, build_instance, config
    from paper_1812_07152_b200.distributed import column_shard

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.device is not None:  # testing the N>1 path on fewer GPUs (ranks share a device)
        local = args.device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spec, q_total = config(args.config)
    if args.q:
        q_total = args.q
    if world > 1:  # every rank builds the same CDS: share the host cores instead of oversubscribing them
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        spec.threads = max(1, (os.cpu_count() or 1) // local_world)
    t0 = time.time()
    inst = build_instance(spec)
    cds = inst.cds
    log(f"[rank {rank}] built {args.config} in {time.time() - t0:.1f}s: near={cds.num_near} far={cds.num_far} "
        f"|D|={cds.d_elems} |B|={cds.b_elems} |V|={cds.v_elems}")
    c0, c1 = column_shard(q_total, world, rank)
    q = c1 - c0
    ev = Evaluator(cds, devices=(local,))
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    w = torch.randn((q, cds.n), dtype=torch.float64, device=dev, generator=gen)  # n x q column major
    y = torch.empty_like(w)
    stream = torch.cuda.Stream(device=dev)
    l2_small = (w.numel() * 8 + cds.bytes(0)) < 4 * 126e6
    flush = torch.empty(int(256e6 // 4), dtype=torch.float32, device=dev) if l2_small else None

    def step(time_phases=False):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=stream.cuda_stream, time_phases=time_phases)

    # warm up with the same graph the timed steps replay (captured with per-launch events)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(time_phases=True)
    torch.cuda.synchronize()

    # ---- device-resident timed region
    phase_ms = None
    step_ms = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(time_phases=True)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            ph = ev.phases()
            if phase_ms is None:
                phase_ms = [0.0] * len(ph)
                phase_info = ph
            for i, p in enumerate(ph):
                phase_ms[i] += p["ms"]
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.summary()
    local_ms = sum(step_ms)
    total_ms = allmax(local_ms)
    ms_per_step = total_ms / args.steps
    flops_step = cds.flops(q_total)
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # dominant kernel: the launch with the largest share of the step (the DAG launch)
    shares = [m / local_ms for m in phase_ms]
    dom = max(range(len(phase_ms)), key=lambda i: phase_ms[i])
    pinfo = phase_info[dom]
    dom_ms = phase_ms[dom] / args.steps
    dom_flops = pinfo["flops_per_col"] * q
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json"), {}) or {}
    traffic = (prof.get(args.config) or {}).get("dominant_dram_bytes_per_launch")
    kname = {"dag": "eval_dag (every GEMM tile of every tree level)"}.get(pinfo["kind"], f"{pinfo['kind']} L{pinfo['level']}")
    roofline = {"bound": "tensor", "achieved": dom_flops / (dom_ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": dom_flops / (dom_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                "traffic": traffic, "kernel": kname, "share_of_step": shares[dom],
                "peak_source": "measured FP64 DMMA peak on this pool (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "algorithmic_flops_per_launch": dom_flops,
                # the bases' unit rows are row copies, not multiply-adds: the kernel's flops
                # above exclude them; `value` counts the reference's 2Q(2|V|+|B|+|D|)
                "identity_row_flops_not_executed": max(0.0, flops_step / world - sum(p["flops_per_col"] for p in phase_info) * q),
                "algorithmic_bytes_per_launch": pinfo["gen_bytes"] + pinfo["io_bytes_per_col"] * q}
    # diagnostic (untimed): the same evaluation as level-by-level launches, per-launch times
    with torch.cuda.stream(stream):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=stream.cuda_stream, time_phases=True, graph=False,
                           levels=True)
    torch.cuda.synchronize()
    level_phases = [{"kind": p["kind"], "level": p["level"], "ms": round(p["ms"], 4),
                     "tflops": round(p["flops_per_col"] * q / max(p["ms"], 1e-9) / 1e9, 2)} for p in ev.phases()]
    # whole-evaluation roofline: max(flops / P_fp64, bytes / HBM)
    # The bound counts the flops the evaluation executes: the interpolative bases' unit rows
    # are row copies (identity rows), so the reference's 2Q(2|V|+|B|+|D|), which
    # `value` keeps, can exceed what a B200 must multiply; frac_reference_flops shows that.
    exec_flops = sum(p["flops_per_col"] for p in phase_info) * q
    t_bytes = cds.bytes(q) / (hbm_peak() * 1e9)
    t_roof = max(exec_flops / (FP64_PEAK_TFLOPS * 1e12), t_bytes)
    t_roof_ref = max(flops_step / world / (FP64_PEAK_TFLOPS * 1e12), t_bytes)
    eval_roofline = {"time_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms_per_step,
                     "bound": "fp64" if exec_flops / (FP64_PEAK_TFLOPS * 1e12) >= t_bytes else "hbm",
                     "executed_flops_per_step": exec_flops,
                     "frac_reference_flops": t_roof_ref * 1e3 / ms_per_step}
    launches = ev.info().launches_per_eval * args.steps
    phases_out = [{"kind": p["kind"], "level": p["level"], "ms": round(m / args.steps, 4)}
                  for p, m in zip(phase_info, phase_ms)]

    # ---- end to end through the C-ABI with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        wh = torch.empty((q, cds.n), dtype=torch.float64, pin_memory=True)
        wh.copy_(w)
        yh = torch.empty((q, cds.n), dtype=torch.float64, pin_memory=True)
        ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)  # warm-up (allocates staging)
        st = EvalStats()
        barrier()
        t_e = time.perf_counter()
        for _ in range(args.e2e_steps):
            ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q, stats=st)
        e2e_s = allmax(time.perf_counter() - t_e) / args.e2e_steps
        ok = bool(torch.equal(yh, y.cpu()))
        e2e = {"value": flops_step / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * cds.n * q_total,
               "d2h_bytes_per_step": 8 * cds.n * q_total, "ms_per_step": e2e_s * 1e3, "steps": args.e2e_steps,
               "matches_device_path_bitwise": ok}
        del wh, yh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = run_reference(args.config, 1, 0, args.cpu_step_s, os.cpu_count() or 1, timeout=120.0)
        if "error" not in res:
            v = res["flops_per_step"] / statistics.mean(res["times"]) / 1e9
            cpu = {"value": v, "unit": "GFLOP/s", "cores": res["threads"], "kind": "reference",
                   "sample": f"{res['q']} of {q_total} W columns of the same CDS, 1 timed evaluate "
                             f"(cost linear in Q); reference hmx::evaluate built -O3 -DNDEBUG",
                   "cpu": cpu_model(), "retries": res["attempts"]}
        else:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "failed: " + res["error"]}

    clk_all = [clk]
    if world > 1:
        clk_all = [None] * world
        dist.all_gather_object(clk_all, clk)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded points (repo builder, seed 42), W ~ N(0,1); the paper's datasets are absent",
            "config": {"workload": DESCR.get(args.config, args.config), "name": args.config, "n": cds.n,
                       "q_total": q_total, "q_per_gpu": q, "parallelism": f"column-shard x{world} (CDS replicated)",
                       "l2": ("inputs larger than L2 (W %.2f GB/GPU, CDS %.2f GB)" % (8 * cds.n * q / 1e9,
                              8 * (cds.d_elems + cds.b_elems + cds.v_elems) / 1e9)) if flush is None
                             else "L2 flushed (256 MB write) between timed steps",
                       "cds": {"near": cds.num_near, "far": cds.num_far, "leaves": int(len(cds.leaves())),
                               "D": cds.d_elems, "B": cds.b_elems, "V": cds.v_elems,
                               "max_srank": int(cds.sranks.max())}},
            "roofline": roofline,
            "eval_roofline": eval_roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": {"sm_mhz": clk_all[0]["sm_mhz"], "sm_max_mhz": clk_all[0]["sm_max_mhz"],
                       "reasons": sorted({r for c in clk_all for r in c["reasons"]})},
            "phases_ms": phases_out,
            "level_launch_breakdown": level_phases,
        }
        print(json.dumps(line), flush=True)
    ev.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "reference-child"])
    ap.add_argument("--config", default="cfg5-hss")
    ap.add_argument("--q", type=int, default=0, help="override the config's total column count")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-step-s", type=float, default=8.0, help="target seconds of the cpu_baseline sample")
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="target seconds per reference-arm step")
    ap.add_argument("--ref-threads", type=int, default=1)
    ap.add_argument("--ref-steps", type=int, default=1)
    ap.add_argument("--ref-warmup", type=int, default=0)
    ap.add_argument("--ref-cols", type=int, default=0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --device: exercise the N>1 path with ranks sharing one GPU (testing only)")
    ap.add_argument("--device", type=int, default=None, help="override LOCAL_RANK's device (testing only)")
    args = ap.parse_args()
    if args.impl == "reference-child":
        args.ref_step_s = args.ref_step_s
        reference_child(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
