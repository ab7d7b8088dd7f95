#!/bin/bash
# End-of-round evidence on the GPU box (gpurun, repo root): tag = first argument.
#   GPU tests, the default bench line (all legs) and the reference arm, an ncu launch list of
#   the bench's matvec steps, one ncu --set full capture of the tensor-core kernel, trace stats.
T=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cg --no-extra --no-cpu \
  > gpurun_out/${T}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmatvec_tc -s 3 -c 1 \
  -o gpurun_out/${T}_kmatvec_tc -f python bench.py --steps 2 --warmup 3 --no-cg --no-extra --no-cpu \
  > gpurun_out/${T}_ncu_full.log 2>&1
TRACE=1 timeout 300 python tools/probes/gpu_trace_stats.py > gpurun_out/${T}_trace.log 2>&1
tail -3 gpurun_out/${T}_gputests.log
cut -c1-400 gpurun_out/${T}_bench.json
