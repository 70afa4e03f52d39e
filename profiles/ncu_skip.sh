mkdir -p gpurun_out
SKR_SKIP_MATH=1 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg -k regex:attn_bwd_kernel -c 1 python profiles/trace_bwd.py 64 > gpurun_out/ncu_skip.txt 2>&1
ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg -k regex:attn_bwd_kernel -c 1 python profiles/trace_bwd.py 64 > gpurun_out/ncu_noskip.txt 2>&1
grep -E "sm__pipe|gpu__time|issue_active|cycles_active" gpurun_out/ncu_skip.txt gpurun_out/ncu_noskip.txt
