#!/bin/bash
# A/B of kernel variants, interleaved over REPS repetitions (kernel-only time at every trace
# shape, no trace), then the operator error of each variant once.
T=${1:-ab}
REPS=${REPS:-2}
for rep in $(seq $REPS); do
  for lib in base probe_libs/*.so; do
    name=$(basename $lib .so)
    if [ "$lib" = base ]; then unset WGP_LIB_PATH; else export WGP_LIB_PATH=$PWD/$lib; fi
    echo "=== $name rep $rep" >> gpurun_out/${T}.log
    TRACE=0 timeout 300 python tools/probes/gpu_trace_stats.py >> gpurun_out/${T}.log 2>&1
  done
done
for lib in base probe_libs/*.so; do
  name=$(basename $lib .so)
  if [ "$lib" = base ]; then unset WGP_LIB_PATH; else export WGP_LIB_PATH=$PWD/$lib; fi
  echo "=== $name acc" >> gpurun_out/${T}.log
  timeout 300 python tools/probes/ab_acc.py >> gpurun_out/${T}.log 2>&1
done
cat gpurun_out/${T}.log
