#!/bin/bash
# knob sweep for narrow DAGs on one box (device-resident probe; each run a fresh process)
mkdir -p gpurun_out
out=gpurun_out/sweep.txt; : > $out
for cs in 1 32; do for sp in 1 2 4; do
  echo "CSTRIDE=$cs COLSPLIT=$sp $(HMXG_CSTRIDE=$cs HMXG_COLSPLIT=$sp python tools/probe.py ${CFGS:-cfg1-hss} 2>&1 | grep DAG | tr '\n' ' ')" >> $out
done; done
for cs in 1 32; do
  HMXG_CSTRIDE=$cs HMXG_COLSPLIT=${SP:-4} HMXG_LIBRARY=build_ab/libhmxg_trace.so python tools/dag_trace.py cfg1-hss > gpurun_out/trace_cfg1_cs$cs.txt 2>&1
done
cat $out; tail -15 gpurun_out/trace_cfg1_cs*.txt
