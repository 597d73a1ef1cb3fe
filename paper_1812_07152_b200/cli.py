"""``hmx``-compatible command line for the B200 evaluator (proj/tools/hmx.cpp).

    python -m paper_1812_07152_b200 eval --out DIR [--w W.bin | --q Q --seed S] [--y Y.bin]
    python -m paper_1812_07152_b200 inspect --n N --d D [--synth uniform] ... --out DIR
    python -m paper_1812_07152_b200 bench --out DIR --q-list 1 256 1024
    python -m paper_1812_07152_b200 accuracy --n N --bacc-list 1e-2 1e-3 1e-5 --q Q

``eval`` is ``cmd_eval`` (hmx.cpp:141-155) on the GPU: it reads ``DIR/hmat.cds`` (written
by the reference's ``hmx inspect`` or by ``inspect`` here), takes W from ``--w`` or the
reference's seeded random W (bit-identical, hmx.cpp:117-122), evaluates Y = K~ W on the
B200 and writes ``--y``. ``plan.json`` is read when present (its lowering switches only
pick a CPU schedule, so the GPU result does not depend on it); the reference requires it.
``inspect`` runs this repo's native instance builder (not the reference inspector) and
writes ``hmat.cds`` + ``plan.json``. ``bench`` times the evaluation of a stored CDS for
each Q on the device (W/Y resident in HBM) and end to end (host buffers). ``accuracy`` is
``cmd_accuracy`` (hmx.cpp:157-170, accuracy_sweep pipeline.cpp:256-287): per bacc it builds
the CDS (this repo's builder), evaluates on the B200 and measures eps_f with the GPU error
oracle (dense for n <= 16384, else 256 sampled rows), printing the reference's CSV.

The common options of hmx.cpp:39-58 are accepted with the same names; exit codes follow
hmx.cpp:12-16 (0 ok, 2 usage, 3 I/O, 5 numeric guard, 1 other).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_NUMERIC_GUARD = 0, 2, 3, 5


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 2 like CLI11 parse errors (hmx.cpp:271-274)
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def _add_common(p: argparse.ArgumentParser) -> None:
    """CommonOpts (hmx.cpp:18-58), same defaults."""
    p.add_argument("--points", default="")
    p.add_argument("--format", default="auto", choices=["csv", "bin", "auto"])
    p.add_argument("--synth", default="")
    p.add_argument("--n", type=int, default=4096)
    p.add_argument("--d", type=int, default=2)
    p.add_argument("--mode", default="hss")
    p.add_argument("--leaf", type=int, default=256)
    p.add_argument("--kernel", default="gaussian:1.0")
    p.add_argument("--bacc", type=float, default=1e-5)
    p.add_argument("--max-rank", type=int, default=256)
    p.add_argument("--agg", type=int, default=2)
    p.add_argument("--sampling-size", type=int, default=32)
    p.add_argument("--workers", type=int, default=0)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default="hmx_out")
    p.add_argument("--exact-sampling", action="store_true")
    p.add_argument("--near-blocksize", type=int, default=2)
    p.add_argument("--far-blocksize", type=int, default=4)
    p.add_argument("--device", type=int, default=0, help="CUDA device (B200 addition)")


def _echo_config(cmd: str, o, n: int, d: int) -> None:
    """echo_config (hmx.cpp:104-115)."""
    src = f" points={o.points}" if o.points else " synth=" + (o.synth or "uniform")
    workers = o.workers or (os.cpu_count() or 1)
    print(f"config: cmd={cmd} n={n} d={d}{src} mode={o.mode} leaf={o.leaf} kernel={o.kernel}"
          f" bacc={o.bacc:g} max_rank={o.max_rank} agg={o.agg} sampling_size={o.sampling_size}"
          f" near_blocksize={o.near_blocksize} far_blocksize={o.far_blocksize} workers={workers}"
          f" seed={o.seed} exact_sampling={1 if o.exact_sampling else 0} out={o.out}")


def _load_stored(o):
    from .executor import EvalPlan
    from .serial import CdsFile, load_plan

    f = CdsFile(os.path.join(o.out, "hmat.cds"))
    plan_path = os.path.join(o.out, "plan.json")
    plan = load_plan(plan_path) if os.path.exists(plan_path) else EvalPlan(p=os.cpu_count() or 1)
    if o.workers:
        plan.p = o.workers
    return f, plan


def cmd_eval(o) -> int:
    from .executor import EvalStats, Evaluator
    from .serial import load_matrix, random_w, save_matrix

    _echo_config("eval", o, 0, 0)
    f, plan = _load_stored(o)
    cds = f.cds
    w = load_matrix(o.w) if o.w else random_w(cds.n, o.q, o.seed)
    if w.shape[0] != cds.n:
        raise ValueError("evaluate: W row count does not match the point count")
    ev = Evaluator(cds, devices=(o.device,))
    stats = EvalStats()
    t0 = time.perf_counter()
    y = ev.evaluate(w, stats) if w.shape[1] else np.zeros((cds.n, 0), order="F")
    seconds = time.perf_counter() - t0
    print(f"eval: n={cds.n} q={w.shape[1]} workers={plan.p} time={seconds:g}s locked_pairs={stats.locked_pairs}"
          f" device_ms={stats.device_ms:.4f}")
    if o.y:
        save_matrix(o.y, y)
    ev.close()
    f.close()
    return EXIT_OK


def _builder_spec(o):
    from .instance import EXACT_SAMPLING, InstanceSpec

    if o.points:
        raise ValueError("inspect: --points files are not supported by the B200 builder; use --synth")
    synth = o.synth or "uniform"
    if synth not in ("uniform", "grid2d", "mixture", "normal", "quantized"):
        raise ValueError(f"inspect: unsupported --synth {synth}")
    spec = InstanceSpec(n=o.n, d=2 if synth == "grid2d" else o.d, points=synth, seed=o.seed, leaf=o.leaf,
                        max_rank=o.max_rank, tol=o.bacc, knn_k=o.sampling_size,
                        near_blocksize=o.near_blocksize, far_blocksize=o.far_blocksize,
                        coarsen_agg=o.agg, coarsen_p=o.workers or (os.cpu_count() or 1),
                        sample_rows=EXACT_SAMPLING if o.exact_sampling else 0)
    if o.mode == "hss":
        spec.mode = "hss"
    elif o.mode.startswith("tau:"):
        spec.mode, spec.tau = "tau", float(o.mode[4:])
    elif o.mode.startswith("budget:"):
        spec.mode, spec.budget = "budget", float(o.mode[7:])
    else:
        raise ValueError("bad --mode, expected hss or tau:VALUE")
    if o.kernel.startswith("gaussian:"):
        spec.kernel, spec.h = "gaussian", float(o.kernel[9:])
    elif o.kernel.startswith("exponential:"):
        spec.kernel, spec.h = "exponential", float(o.kernel[12:])
    elif o.kernel == "invdist":
        spec.kernel = "invdist"
    else:
        raise ValueError("bad --kernel, expected gaussian:H or invdist")
    return spec


def cmd_inspect(o) -> int:
    import json

    from .executor import generate_plan
    from .instance import build_instance
    from .serial import IoError, save_cds

    spec = _builder_spec(o)
    _echo_config("inspect", o, spec.n, spec.d)
    t0 = time.perf_counter()
    inst = build_instance(spec)
    cds = inst.cds
    os.makedirs(o.out, exist_ok=True)
    save_cds(os.path.join(o.out, "hmat.cds"), cds, dim=spec.d, bacc=o.bacc, max_rank=o.max_rank,
             leaf_size=o.leaf)
    plan = generate_plan(cds)
    try:
        with open(os.path.join(o.out, "plan.json"), "w") as fh:
            json.dump({k: getattr(plan, k) for k in ("block_lowering_near", "block_lowering_far", "coarsen_lowering",
                                                     "peel_top", "p", "block_threshold", "coarsen_threshold")},
                      fh, indent=2)
            fh.write("\n")
    except OSError as e:
        raise IoError(str(e)) from e
    print(f"p1: nodes={cds.num_nodes} height={cds.height} near_pairs={cds.num_near} far_pairs={cds.num_far}")
    print(f"p2: max_srank={int(cds.sranks.max()) if cds.num_nodes else 0} dgen={cds.dgen.size}"
          f" bgen={cds.bgen.size} vgen={cds.vgen.size} time={time.perf_counter() - t0:g}s")
    inst.close()
    return EXIT_OK


def cmd_bench(o) -> int:
    import torch

    from .executor import Evaluator
    from .serial import random_w

    _echo_config("bench", o, 0, 0)
    f, _ = _load_stored(o)
    cds = f.cds
    ev = Evaluator(cds, devices=(o.device,))
    dev = torch.device("cuda", o.device)
    stream = torch.cuda.Stream(dev)
    print("q,device_seconds,e2e_seconds,tflops_device")
    for q in o.q_list:
        w = random_w(cds.n, q, o.seed)
        y = np.empty_like(w, order="F")
        wd = torch.from_numpy(w.T.copy()).to(dev)
        yd = torch.empty_like(wd)
        with torch.cuda.stream(stream):
            for _ in range(3):
                ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record(stream)
            for _ in range(reps):
                ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=stream.cuda_stream)
            e1.record(stream)
        stream.synchronize()
        dev_s = e0.elapsed_time(e1) / 1e3 / reps
        ev.evaluate(w, out=y)
        t0 = time.perf_counter()
        for _ in range(3):
            ev.evaluate(w, out=y)
        e2e_s = (time.perf_counter() - t0) / 3
        print(f"{q},{dev_s:.6g},{e2e_s:.6g},{cds.flops(q) / dev_s / 1e12:.4g}")
    ev.close()
    f.close()
    return EXIT_OK


def cmd_accuracy(o) -> int:
    from .accuracy import DevicePoints, ErrorMode, Kernel
    from .executor import EvalStats, Evaluator
    from .instance import build_instance
    from .serial import random_w

    t_start = time.perf_counter()
    spec = _builder_spec(o)
    _echo_config("accuracy", o, spec.n, spec.d)
    kernel = Kernel(spec.kernel, spec.h)
    mode = ErrorMode.DENSE if spec.n <= 16384 else ErrorMode.SAMPLED
    w = random_w(spec.n, o.q, o.seed)
    lines, p1_seconds, oracle_seconds, dp = ["bacc,eps_f,eval_seconds,p2_seconds"], 0.0, 0.0, None
    for i, bacc in enumerate(o.bacc_list):
        spec.tol = bacc
        inst = build_instance(spec)
        st = inst.stats
        p1 = st["seconds_points"] + st["seconds_tree"] + st["seconds_interactions"] + st["seconds_sampling"]
        if i == 0:
            p1_seconds = p1
            dp = DevicePoints(inst.points(), kernel, o.device)
        ev = Evaluator(inst.cds, devices=(o.device,))
        stats = EvalStats()
        y = ev.evaluate(w, stats)
        t0 = time.perf_counter()
        eps = dp.relative_error_vs(y, w, mode, o.seed)
        oracle_seconds += time.perf_counter() - t0
        lines.append(f"{bacc:g},{eps:g},{stats.seconds:g},{st['seconds_total'] - p1:g}")
        ev.close()
        inst.close()
    print("\n".join(lines))
    print(f"# p1={p1_seconds:g}s oracle={oracle_seconds:g}s total={time.perf_counter() - t_start:g}s")
    if dp is not None:
        dp.close()
    return EXIT_OK


def main(argv=None) -> int:
    from .accuracy import NumericGuardError
    from .serial import IoError

    app = _Parser(prog="hmx-b200", description="B200 evaluation of hierarchical kernel matrices")
    sub = app.add_subparsers(dest="cmd", parser_class=_Parser)
    p_inspect = sub.add_parser("inspect", help="build a CDS with the native builder, write hmat.cds")
    _add_common(p_inspect)
    p_eval = sub.add_parser("eval", help="multiply a stored matrix by W on the B200")
    _add_common(p_eval)
    p_eval.add_argument("--w", default="")
    p_eval.add_argument("--q", type=int, default=16)
    p_eval.add_argument("--y", default="")
    p_bench = sub.add_parser("bench", help="device and end-to-end evaluation time per Q")
    _add_common(p_bench)
    p_bench.add_argument("--q-list", type=int, nargs="+", default=[1, 256, 1024, 2048])
    p_acc = sub.add_parser("accuracy", help="bacc sweep with the GPU error oracle, CSV output")
    _add_common(p_acc)
    p_acc.add_argument("--bacc-list", type=float, nargs="+", default=[1e-2, 1e-3, 1e-5])
    p_acc.add_argument("--q", type=int, default=16)
    try:
        o = app.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    if o.cmd is None:
        app.print_usage(sys.stderr)
        return EXIT_USAGE
    try:
        return {"eval": cmd_eval, "inspect": cmd_inspect, "bench": cmd_bench, "accuracy": cmd_accuracy}[o.cmd](o)
    except IoError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except NumericGuardError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NUMERIC_GUARD
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001 - the CLI's catch-all (hmx.cpp:292-295)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
