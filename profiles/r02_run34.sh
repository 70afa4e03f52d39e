# Round 2 (session 3), GPU call 34: ncu --set full (with source) of the d = 64 kernels on C2 (configs[1]),
# the final build, for the source-level stall attribution of the d = 64 forward.
mkdir -p gpurun_out/r02e_c2
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config C2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_c2/launches.csv $CMD > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/r02e_c2/prof_fwd $CMD > gpurun_out/r34_prof_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/r02e_c2/prof_bwd $CMD > gpurun_out/r34_prof_bwd.log 2>&1
ls -la gpurun_out/r02e_c2
