#!/bin/bash
# FP64 pipe-sharing probe, cfg1/cfg2 device timings and a cfg1 item trace
mkdir -p gpurun_out
./tools/fp64_mix > gpurun_out/fp64_mix.txt 2>&1
python tools/probe.py cfg1-hss cfg2-h2b > gpurun_out/probe_small.txt 2>&1
HMXG_LIBRARY=build_ab/libhmxg_trace.so python tools/dag_trace.py cfg1-hss > gpurun_out/trace_cfg1.txt 2>&1
timeout 600 python bench.py --config cfg1-hss --steps 20 --warmup 5 --e2e-steps 3 --dropin-steps 2 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
cat gpurun_out/fp64_mix.txt; grep -E "DAG|dag|gather|scatter" gpurun_out/probe_small.txt; tail -n 25 gpurun_out/trace_cfg1.txt
