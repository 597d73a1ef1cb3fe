#!/bin/bash
# A/B of several builds on one box (dev tool): tools/ab_libs.sh "CFGS" LIB... -> device-resident probe, twice each
CFGS=${1:-cfg1-hss}; shift
for rep in 1 2; do
  echo "base $(python tools/probe.py $CFGS 2>&1 | grep ' DAG ' | tr '\n' ' ')"
  for L in "$@"; do echo "$L $(HMXG_LIBRARY=$L python tools/probe.py $CFGS 2>&1 | grep ' DAG ' | tr '\n' ' ')"; done
done
