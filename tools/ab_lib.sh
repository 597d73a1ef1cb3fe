#!/bin/bash
# A/B of two builds on one box (dev tool): tools/ab_lib.sh LIB_B "cfg..." -> device-resident probe
# of the in-tree libhmxg.so and LIB_B, twice each, interleaved
mkdir -p gpurun_out
B=${1:?lib}; CFGS=${2:-"cfg1-hss cfg2-h2b cfg5-hss"}
for rep in 1 2; do
  echo "A $(python tools/probe.py $CFGS 2>&1 | grep 'DAG' | tr '\n' ' ')"
  echo "B $(HMXG_LIBRARY=$B python tools/probe.py $CFGS 2>&1 | grep 'DAG' | tr '\n' ' ')"
done
