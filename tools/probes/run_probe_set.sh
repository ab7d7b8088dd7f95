#!/bin/bash
# GPU probe batch (run through gpurun from the repo root): tag = first argument.
# Each step is bounded by its own timeout; outputs land in gpurun_out/<tag>_*.log.
T=${1:-p}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1
timeout 900 python tools/probes/gpu_probe_anchor.py c2 c4 c3 > gpurun_out/${T}_anchor_new.log 2>&1
WGP_LIB_PATH=tools/probes/_variants/libwarmgp_kexp.so timeout 600 python tools/probes/gpu_probe_anchor.py c2 c3 > gpurun_out/${T}_anchor_kexp.log 2>&1
timeout 300 python tools/probes/gpu_probe_kerr.py > gpurun_out/${T}_kerr_new.log 2>&1
WGP_LIB_PATH=tools/probes/_variants/libwarmgp_kexp.so timeout 300 python tools/probes/gpu_probe_kerr.py > gpurun_out/${T}_kerr_kexp.log 2>&1
timeout 300 python tools/probes/gpu_probe_tc_shapes.py > gpurun_out/${T}_shapes_new.log 2>&1
WGP_LIB_PATH=tools/probes/_variants/libwarmgp_kexp.so timeout 300 python tools/probes/gpu_probe_tc_shapes.py > gpurun_out/${T}_shapes_kexp.log 2>&1
tail -3 gpurun_out/${T}_gputests.log
