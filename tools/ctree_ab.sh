#!/bin/bash
# CTree A/B on one box (dev tool): cfg1 device-resident DAG vs HMXG_CTREE=1 per cluster size, and
# a CTree item trace with per-level and per-block stamps (needs build_ab/libhmxg_trace.so, a
# -DHMXG_TRACE build)
mkdir -p gpurun_out
echo "DAG $(python tools/probe.py cfg1-hss 2>&1 | grep DAG)" > gpurun_out/ctree_ab.txt
for cs in 2 4 8; do echo "CTree C=$cs $(HMXG_CTREE=1 HMXG_CT_CLUSTER=$cs python tools/probe.py cfg1-hss 2>&1 | grep DAG)" >> gpurun_out/ctree_ab.txt; done
[ -f build_ab/libhmxg_trace.so ] && HMXG_CTREE=1 HMXG_CT_CLUSTER=8 HMXG_LIBRARY=build_ab/libhmxg_trace.so python tools/dag_trace.py cfg1-hss > gpurun_out/ctree_trace.txt 2>&1
cat gpurun_out/ctree_ab.txt
