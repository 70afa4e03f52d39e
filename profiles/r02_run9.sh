# Round 2, GPU call 9: what FlashAttention-4's d = 128 forward does differently (context library,
# same packed S4n1 batch): per-launch cycles, instructions, pipe utilisation, launch shape -- next to
# this build's forward under the same metric set.
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__block_size,launch__grid_size,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"cutlass|[Ff]lash|fmha|Sm100" -c 6 --csv --log-file gpurun_out/r9_fa4_s4n1.csv python tools/comparators.py --config S4n1 --impls fa4 --reps 1 > gpurun_out/r9_fa4.log 2>&1
ls gpurun_out | grep r9
