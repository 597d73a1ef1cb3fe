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
# Configs the reference's own inspector supports (HSS mode: interaction.cpp:115-143 has no
# budget mode). For them the reference arm builds its CDS through the reference's own public
# pipeline in oracle/_ref (tst::make_instance: synth_points, build_cluster_tree,
# compute_interactions(Hss), build_samples, compress, blocking, coarsening, build_cds) and
# evaluates it with the stock plan (hmx::generate_plan); none of this repo's libraries is
# loaded in that process. Other configs read a CDS file the repo builder wrote (hmat.cds,
# via hmx::load_cds).
REF_SPECS = {
    "cfg1-hss": dict(n=4096, d=3, shape=1, mode=1, leaf=128, h=0.5, bacc=1e-5, max_rank=64, seed=42),
    "cfg5-hss": dict(n=262144, d=3, shape=1, mode=1, leaf=256, h=0.1, bacc=1e-6, max_rank=128, seed=42),
}


def cpu_info() -> dict:
    """`lscpu`-style facts for the CPU line: model, logical CPUs, the SIMD flags that matter."""
    model, flags = "unknown", set()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model == "unknown":
                model = line.split(":", 1)[1].strip()
            elif line.startswith("flags") and not flags:
                flags = set(line.split(":", 1)[1].split())
    except Exception:
        pass
    keep = [f for f in ("sse4_2", "avx", "avx2", "fma", "avx512f", "avx512dq", "avx512vl", "amx_tile") if f in flags]
    return {"model": model, "logical_cpus": os.cpu_count(), "flags": keep}


def reference_child(args) -> None:
    """Runs in a forked child: the reference hmx::evaluate (oracle/_ref) on a column slice,
    with args.ref_threads workers, then the same slice's first columns at p = 1, compared bit
    for bit (the WorkerPool race F5 must not have changed the result)."""
    import numpy as np

    import oracle

    threads = max(1, args.ref_threads)
    t0 = time.time()
    if args.config in REF_SPECS and not args.cds_file:
        src = oracle.RefInstance(oracle.RefInstanceSpec(**REF_SPECS[args.config], p=threads))
        bits = src.generate_plan(threads)
        run = lambda w, p: src.evaluate_timed(w, bits, p)  # noqa: E731
        source = ("reference inspector (oracle/_ref tst::make_instance pipeline: synth_points, build_cluster_tree, "
                  "compute_interactions(Hss), build_samples, compress, blocking, coarsening, build_cds); "
                  "stock plan hmx::generate_plan")
    else:
        src = oracle.RefCds.load(args.cds_file)  # hmx::load_cds (serial.cpp:299-308)
        bits = 0
        run = lambda w, p: src.evaluate(w, p=p, plan_bits=bits)  # noqa: E731
        source = "repo builder CDS written as hmat.cds, read by hmx::load_cds (the reference has no budget mode)"
    build_s = time.time() - t0
    cds = src.cds
    n = cds.n
    rng = np.random.default_rng(1234)
    q = args.ref_cols
    if q <= 0:  # calibrate: aim for ~args.ref_step_s seconds per step
        wq = np.asfortranarray(rng.standard_normal((n, 8)))
        _, sec = run(wq, threads)
        rate = cds.flops(8) / max(sec, 1e-6)
        q = int(min(args.q_total, max(8, args.ref_step_s * rate / cds.flops(1))))
    w = np.asfortranarray(rng.standard_normal((n, q)))
    times = []
    y = None
    for it in range(args.ref_warmup + args.ref_steps):
        y, sec = run(w, threads)  # EvalStats.seconds (executor.cpp:276,289-294)
        if it >= args.ref_warmup:
            times.append(sec)
    q1 = min(q, 8)
    y1, sec1 = run(np.asfortranarray(w[:, :q1]), 1)
    print(json.dumps({"q": q, "threads": threads, "times": times, "flops_per_step": cds.flops(q),
                      "flops_per_col": cds.flops(1), "plan_bits": bits, "source": source, "build_s": build_s,
                      "p1": {"q": q1, "seconds": sec1, "gflops": cds.flops(q1) / max(sec1, 1e-9) / 1e9,
                             "bitwise_equal_to_p": bool(np.array_equal(y1, y[:, :q1]))},
                      "cds": {"n": n, "near": cds.num_near, "far": cds.num_far, "D": cds.d_elems, "B": cds.b_elems,
                              "V": cds.v_elems}}), flush=True)


def write_cds_child(args) -> None:
    """Builds a config with the repo builder and writes it as hmat.cds (configs the reference
    inspector cannot build; run in its own process, before the reference child)."""
    from paper_1812_07152_b200 import build_instance, config, serial

    spec, _ = config(args.config)
    inst = build_instance(spec)
    serial.save_cds(args.cds_file, inst.cds, dim=spec.d, bacc=spec.tol, max_rank=spec.max_rank)


def run_reference(config_name: str, steps: int, warmup: int, step_s: float, threads: int, timeout: float):
    """The reference in a watchdog child; retries a hang/crash, then falls back to p = 1."""
    from paper_1812_07152_b200 import config

    _, q_total = config(config_name)
    attempts = []
    cds_file = ""
    tmpdir = None
    if config_name not in REF_SPECS:
        tmpdir = tempfile.mkdtemp(prefix="hmx_ref_")
        cds_file = os.path.join(tmpdir, "hmat.cds")
        subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "write-cds", "--config", config_name,
                        "--cds-file", cds_file], check=True, timeout=1800)
    try:
        for p in (threads, threads, 1):
            cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference-child", "--config", config_name,
                   "--ref-threads", str(p), "--ref-steps", str(steps), "--ref-warmup", str(warmup),
                   "--ref-step-s", str(step_s), "--q-total", str(q_total)]
            if cds_file:
                cmd += ["--cds-file", cds_file]
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
            except subprocess.TimeoutExpired:
                attempts.append(f"p={p}: hang (killed after {timeout:.0f}s)")
                continue
            if out.returncode != 0:
                attempts.append(f"p={p}: exit {out.returncode}: {out.stderr.strip()[-200:]}")
                continue
            res = json.loads(out.stdout.strip().splitlines()[-1])
            res["attempts"] = attempts
            return res
        return {"error": "; ".join(attempts)}
    finally:
        if tmpdir:
            import shutil

            shutil.rmtree(tmpdir, ignore_errors=True)


def cpu_baseline_of(res: dict, q_total: int, kind_note: str) -> dict:
    v = res["flops_per_step"] / statistics.mean(res["times"]) / 1e9
    return {"value": v, "unit": "GFLOP/s", "cores": res["threads"], "kind": "reference",
            "sample": (f"{res['q']} of {q_total} W columns per step (cost is linear in Q, SURVEY F8); {kind_note}; "
                       f"CDS: {res['source']}"),
            "cpu": cpu_info(), "retries": res["attempts"], "plan_bits": res["plan_bits"],
            "p1": res["p1"], "cds": res["cds"],
            "build": "oracle/_ref: reference proj/src compiled -O3 -DNDEBUG (shipped Release flags)"}


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1812_07152_b200 import config

    _, q_total = config(args.config)
    threads = os.cpu_count() or 1
    res = run_reference(args.config, args.steps, args.warmup, args.ref_step_s, threads,
                        timeout=max(180.0, 15.0 * (args.steps + args.warmup) * args.ref_step_s + 120.0))
    if "error" in res:
        print(json.dumps({"impl": "reference", "unavailable": "reference evaluate failed: " + res["error"]}))
        return
    t = statistics.mean(res["times"])
    value = res["flops_per_step"] / t / 1e9
    cpu = cpu_baseline_of(res, q_total, f"{args.steps} timed steps after {args.warmup} warm-up")
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)", "impl": "reference",
        "config": {"workload": DESCR.get(args.config, args.config), "name": args.config, "q_sampled": res["q"],
                   "q_total": q_total, "parallelism": f"host threads x{res['threads']}",
                   "same_config": "same BASELINE config; Q sampled (cost exactly linear in Q, SURVEY F8)"},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def measure(args, name, env, steps, warmup, e2e_steps, dropin_steps):
    """Device-resident, end-to-end (pinned) and drop-in (pageable numpy through the Python
    mirror of hmx::evaluate) measurements of one config on this rank's column shard."""
    import numpy as np
    import torch

    from paper_1812_07152_b200 import EvalPlan, EvalStats, Evaluator, build_instance, config, evaluate
    from paper_1812_07152_b200.distributed import column_shard

    rank, world, local, dev, barrier, allmax = (env[k] for k in ("rank", "world", "local", "dev", "barrier", "allmax"))
    spec, q_total = config(name)
    if args.q and name == args.config:
        q_total = args.q
    if world > 1:  # every rank builds the same CDS: share the host cores instead of oversubscribing them
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        spec.threads = max(1, (os.cpu_count() or 1) // local_world)
    t0 = time.time()
    inst = build_instance(spec)
    cds = inst.cds
    log(f"[rank {rank}] built {name} in {time.time() - t0:.1f}s: near={cds.num_near} far={cds.num_far} "
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

    # warm up with the same graph the timed steps replay (captured with per-launch events).
    # A single-launch evaluation (small problems: permutations fused into the DAG launch) is
    # timed without the per-launch event nodes: the step's own events bracket exactly that
    # launch, and on cfg1 the two extra graph nodes cost ~10 us of a ~40 us step.
    with torch.cuda.stream(stream):
        step(time_phases=True)
    torch.cuda.synchronize()
    timed_phases = ev.info().launches_per_eval > 1
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step(time_phases=timed_phases)
    torch.cuda.synchronize()

    # ---- device-resident timed region
    phase_ms = None
    step_ms = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for _ in range(steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(time_phases=timed_phases)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            ph = ev.phases()
            if phase_ms is None:
                phase_ms = [0.0] * len(ph)
                phase_info = ph
            for i, p in enumerate(ph):
                phase_ms[i] += p["ms"] if timed_phases else step_ms[-1]
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.summary()
    # kernels launched inside the timed region: the launches of one timed step (gather, eval_dag,
    # scatter; one fused launch for small problems) x steps -- read before the diagnostic below
    # runs the same evaluation as ~2H+3 per-level launches
    launches = ev.info().launches_per_eval * steps
    local_ms = sum(step_ms)
    total_ms = allmax(local_ms)
    ms_per_step = total_ms / steps
    flops_step = cds.flops(q_total)
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # dominant kernel: the launch with the largest share of the step (the DAG launch)
    shares = [m / local_ms for m in phase_ms]
    dom = max(range(len(phase_ms)), key=lambda i: phase_ms[i])
    pinfo = phase_info[dom]
    dom_ms = phase_ms[dom] / steps
    dom_flops = pinfo["flops_per_col"] * q
    prof = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json"), {}) or {}
    traffic = (prof.get(name) or {}).get("dominant_dram_bytes_per_launch")
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
    phases_out = [{"kind": p["kind"], "level": p["level"], "ms": round(m / steps, 4)}
                  for p, m in zip(phase_info, phase_ms)]

    # ---- end to end through the C-ABI with pinned host buffers
    e2e = None
    y_dev = y.cpu()
    if e2e_steps > 0:
        wh = torch.empty((q, cds.n), dtype=torch.float64, pin_memory=True)
        wh.copy_(w)
        yh = torch.empty((q, cds.n), dtype=torch.float64, pin_memory=True)
        ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)  # warm-up (allocates staging)
        st = EvalStats()
        barrier()
        t_e = time.perf_counter()
        for _ in range(e2e_steps):
            ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q, stats=st)
        e2e_s = allmax(time.perf_counter() - t_e) / e2e_steps
        e2e = {"value": flops_step / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * cds.n * q_total,
               "d2h_bytes_per_step": 8 * cds.n * q_total, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
               "host_buffers": "pinned (torch pin_memory), C-ABI hmxg_evaluate host-pointer path",
               "matches_device_path_bitwise": bool(torch.equal(yh, y_dev))}
        del wh, yh
    ev.close()
    del w, y

    # ---- the drop-in call: paper_1812_07152_b200.evaluate(cds, plan, W) with pageable numpy
    # buffers (the Python mirror of hmx::evaluate; the C++ shim hmx_gpu::evaluate takes the
    # same path with hmx::DenseMatrix). Every call fingerprints the CDS (the resident upload
    # is keyed on its content), stages W / Y through pinned buffers on the host threads.
    dropin = None
    if dropin_steps > 0:
        wn = np.asfortranarray(y_dev.numpy().T)  # any n x q data; y_dev as W keeps host memory low
        yref = None
        evaluate(cds, EvalPlan(), wn, devices=(local,))  # warm-up: upload + staging
        barrier()
        t_d = time.perf_counter()
        for _ in range(dropin_steps):
            yref = evaluate(cds, EvalPlan(), wn, devices=(local,))
        d_s = allmax(time.perf_counter() - t_d) / dropin_steps
        t_f = time.perf_counter()
        cds.fingerprint()
        fp_s = time.perf_counter() - t_f
        dropin = {"value": flops_step / d_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * cds.n * q_total,
                  "d2h_bytes_per_step": 8 * cds.n * q_total, "ms_per_step": d_s * 1e3, "steps": dropin_steps,
                  "fingerprint_ms": fp_s * 1e3,
                  "host_buffers": "pageable numpy (drop-in evaluate(cds, plan, w): content-keyed resident upload, "
                                  "pinned bounce staging on the host threads)"}
        for ev_ in [v[1] for v in cds._cache.values()]:
            ev_.close()
        cds._cache.clear()
        del wn, yref
    out = {
        "value": value, "ms_per_step": ms_per_step, "q_total": q_total, "q": q, "cds": cds, "flush": flush is not None,
        "w_bytes": 8 * cds.n * q, "roofline": roofline, "eval_roofline": eval_roofline, "e2e": e2e,
        "e2e_dropin": dropin, "launches": launches, "clk": clk, "phases_ms": phases_out,
        "level_launch_breakdown": level_phases,
        "cds_info": {"near": cds.num_near, "far": cds.num_far, "leaves": int(len(cds.leaves())), "D": cds.d_elems,
                     "B": cds.b_elems, "V": cds.v_elems, "max_srank": int(cds.sranks.max())},
        "cds_gb": 8 * (cds.d_elems + cds.b_elems + cds.v_elems) / 1e9,
    }
    inst.close()
    return out


def measure_near_otf(args, name, env, steps, warmup):
    """The near field generated on the fly (HMXG_UPLOAD_NEAR_ON_THE_FLY): the config built
    without D on the host, uploaded with points + kernel, every evaluation generating its near
    blocks wave by wave into a bounded scratch. Device-resident, this rank's column shard."""
    import torch

    from paper_1812_07152_b200 import Evaluator, build_instance, config
    from paper_1812_07152_b200.accuracy import Kernel
    from paper_1812_07152_b200.distributed import column_shard

    rank, world, local, dev, barrier, allmax = (env[k] for k in ("rank", "world", "local", "dev", "barrier", "allmax"))
    spec, q_total = config(name)
    spec.skip_near = True
    if world > 1:
        spec.threads = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    inst = build_instance(spec)
    cds = inst.cds
    c0, c1 = column_shard(q_total, world, rank)
    q = c1 - c0
    ev = Evaluator(cds, devices=(local,), points=inst.points(), kernel=Kernel(spec.kernel, spec.h), near_on_the_fly=True)
    w = torch.randn((q, cds.n), dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
    y = torch.empty_like(w)
    stream = torch.cuda.Stream(device=dev)
    for _ in range(warmup):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=stream.cuda_stream, time_phases=True)
    torch.cuda.synchronize()
    barrier()
    ms = []
    gen_ms = leaf_ms = 0.0
    with ClockSampler(local) as clocks:
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=stream.cuda_stream, time_phases=True)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            ph = ev.phases()
            gen_ms += sum(p["ms"] for p in ph if p["kind"] == "near-gen")
            leaf_ms += sum(p["ms"] for p in ph if p["kind"] == "near+leaf")
    ms_step = allmax(sum(ms)) / steps
    waves = sum(1 for p in ev.phases() if p["kind"] == "near-gen")
    out = {"workload": DESCR.get(name, name) + "; near blocks generated on the fly (never resident)",
           "value": cds.flops(q_total) / (ms_step * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_step,
           "q_per_gpu": q, "device_gb": ev.info().device_bytes / 1e9, "near_gb_not_resident": 8 * float(cds.dptr[-1]) / 1e9,
           "waves": waves, "near_gen_ms_per_step": gen_ms / steps, "leaf_waves_ms_per_step": leaf_ms / steps,
           "clocks": clocks.summary()}
    ev.close()
    inst.close()
    return out


def ours(args) -> None:
    import torch
    import torch.distributed as dist

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
        log(f"[rank {rank}] process group up: backend={dist.get_backend()} world={dist.get_world_size()}")

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    env = {"rank": rank, "world": world, "local": local, "dev": dev, "barrier": barrier, "allmax": allmax}
    m = measure(args, args.config, env, args.steps, args.warmup, args.e2e_steps, args.dropin_steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = run_reference(args.config, 1, 0, args.cpu_step_s, os.cpu_count() or 1, timeout=300.0)
        if "error" not in res:
            cpu = cpu_baseline_of(res, m["q_total"], "1 timed evaluate")
        else:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "failed: " + res["error"]}

    # the heavier half of the headline config (BASELINE cfg5 names HSS and H2-b): same
    # measurement, same rank layout, reported under extra
    extra = {}
    # (one GPU only: every rank would build cfg5-H2-b's 18.6 GB near field on the host)
    if args.extra and args.config == "cfg5-hss" and world == 1:
        for xname in args.extra.split(","):
            x = measure(args, xname, env, args.steps, args.warmup, min(args.e2e_steps, 2), min(args.dropin_steps, 1))
            extra[xname.replace("-", "_")] = {
                "workload": DESCR.get(xname, xname), "value": x["value"], "unit": "GFLOP/s",
                "ms_per_step": x["ms_per_step"], "q_per_gpu": x["q"], "roofline": x["roofline"],
                "eval_roofline": x["eval_roofline"], "e2e": x["e2e"], "e2e_dropin": x["e2e_dropin"],
                "gpu_launches": x["launches"], "clocks": x["clk"], "phases_ms": x["phases_ms"], "cds": x["cds_info"],
                "cds_gb": x["cds_gb"]}

    if args.extra and args.config == "cfg5-hss" and args.near_otf and world == 1:
        extra["cfg5_h2b_near_on_the_fly"] = measure_near_otf(args, "cfg5-h2b", env, max(3, args.steps // 2), args.warmup)

    clk_all = [m["clk"]]
    if world > 1:
        clk_all = [None] * world
        dist.all_gather_object(clk_all, m["clk"])
    if rank == 0:
        line = {
            "metric": METRIC, "value": m["value"], "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded points (repo builder, seed 42), W ~ N(0,1); the paper's datasets are absent",
            "config": {"workload": DESCR.get(args.config, args.config), "name": args.config, "n": m["cds"].n,
                       "q_total": m["q_total"], "q_per_gpu": m["q"],
                       "parallelism": f"column-shard x{world} (CDS replicated)",
                       "l2": ("inputs larger than L2 (W %.2f GB/GPU, CDS %.2f GB)" % (m["w_bytes"] / 1e9, m["cds_gb"]))
                             if not m["flush"] else "L2 flushed (256 MB write) between timed steps",
                       "cds": m["cds_info"]},
            "roofline": m["roofline"],
            "eval_roofline": m["eval_roofline"],
            "e2e": m["e2e"],
            "e2e_dropin": m["e2e_dropin"],
            "cpu_baseline": cpu,
            "gpu_launches": m["launches"],
            "clocks": {"sm_mhz": clk_all[0]["sm_mhz"], "sm_max_mhz": clk_all[0]["sm_max_mhz"],
                       "reasons": sorted({r for c in clk_all for r in c["reasons"]})},
            "phases_ms": m["phases_ms"],
            "level_launch_breakdown": m["level_launch_breakdown"],
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "reference-child", "write-cds"])
    ap.add_argument("--config", default="cfg5-hss")
    ap.add_argument("--q", type=int, default=0, help="override the config's total column count")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--dropin-steps", type=int, default=2)
    ap.add_argument("--extra", default="cfg5-h2b", help="comma list of configs measured into `extra` (cfg5-hss runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--near-otf", type=int, default=1, help="measure cfg5-h2b with the near field on the fly (extra)")
    ap.add_argument("--cpu-step-s", type=float, default=8.0, help="target seconds of the cpu_baseline sample")
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="target seconds per reference-arm step")
    ap.add_argument("--ref-threads", type=int, default=1)
    ap.add_argument("--ref-steps", type=int, default=1)
    ap.add_argument("--ref-warmup", type=int, default=0)
    ap.add_argument("--ref-cols", type=int, default=0)
    ap.add_argument("--q-total", type=int, default=2048)
    ap.add_argument("--cds-file", default="")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --device: exercise the N>1 path with ranks sharing one GPU (testing only)")
    ap.add_argument("--device", type=int, default=None, help="override LOCAL_RANK's device (testing only)")
    args = ap.parse_args()
    if args.impl == "reference-child":
        reference_child(args)
    elif args.impl == "write-cds":
        write_cds_child(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
