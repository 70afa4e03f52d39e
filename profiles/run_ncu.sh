#!/bin/bash
# Profiling recipe (B200_PROFILING.md), run under gpurun on ONE GPU:
#   1. launch list of the bench command (cold-cache, serialised per-launch times)
#   2. one `--set full` capture of each attention kernel
# Then, back here: python profiles/summarize_ncu.py --workload C2/n1 --tag r01
CFG=${1:-C2}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config $CFG"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/prof_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/prof_fwd.log 2>&1
ls -la gpurun_out
