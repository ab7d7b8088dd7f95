#!/bin/bash
# Round check on the GPU box (through gpurun, from the repo root): tag = first argument.
#   tests (-m gpu), bench (ours + reference arm), compute-sanitizer on the small workload,
#   ncu launch list of the bench's matvec steps.  Every step bounded by its own timeout.
T=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
if [ "${SANITIZE:-1}" = "1" ]; then
  for tool in racecheck synccheck memcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/probes/sanitize_small.py \
      > gpurun_out/${T}_sanitize_${tool}.log 2>&1
  done
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cg --no-extra --no-cpu \
  > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_gputests.log
cut -c1-300 gpurun_out/${T}_bench.json
