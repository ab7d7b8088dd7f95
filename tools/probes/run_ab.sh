#!/bin/bash
# A/B of tensor-core kernel variants on the GPU box: for each library in probe_libs/ (plus
# the in-tree build as "base"), kernel-only time + per-tile trace stats, and the operator error.
T=${1:-ab}
for lib in base probe_libs/*.so; do
  name=$(basename $lib .so)
  if [ "$lib" = base ]; then unset WGP_LIB_PATH; else export WGP_LIB_PATH=$PWD/$lib; fi
  echo "=== $name" >> gpurun_out/${T}.log
  TRACE=${TRACE:-1} timeout 300 python tools/probes/gpu_trace_stats.py >> gpurun_out/${T}.log 2>&1
  timeout 300 python tools/probes/ab_acc.py >> gpurun_out/${T}.log 2>&1
done
cat gpurun_out/${T}.log
