#!/bin/bash
# A/B on one box: the current libhmxg.so against build_ab/libhmxg_r1.so (round-1 build) on
# cfg5-hss and cfg1-hss (tools/probe.py, device-resident), plus a cfg1 item trace of the
# current kernel (build_ab/libhmxg_trace.so)
mkdir -p gpurun_out
for rep in 1 2; do
  python tools/probe.py cfg5-hss cfg1-hss 2>&1 | grep -E "DAG|dag " > gpurun_out/ab_new_$rep.txt
  HMXG_LIBRARY=build_ab/libhmxg_r1.so python tools/probe.py cfg5-hss cfg1-hss 2>&1 | grep -E "DAG|dag " > gpurun_out/ab_r1_$rep.txt
done
HMXG_LIBRARY=build_ab/libhmxg_trace.so python tools/dag_trace.py cfg1-hss > gpurun_out/trace_cfg1.txt 2>&1
head -50 gpurun_out/ab_*.txt gpurun_out/trace_cfg1.txt
