#!/bin/bash
# two-step schedule model check: run-length sweep on C2 (walls) and walls vs periodic Y
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for run in 64 96 113 120 128 137 160 240; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --run $run >> gpurun_out/ax_runs.jsonl 2>> gpurun_out/ax.err
done
timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --periodic >> gpurun_out/ax_periodic.jsonl 2>> gpurun_out/ax.err
timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast >> gpurun_out/ax_periodic.jsonl 2>> gpurun_out/ax.err
timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --periodic >> gpurun_out/ax_periodic.jsonl 2>> gpurun_out/ax.err
