# Round 2 (session 2), GPU call 10: re-baseline in the new container (bench S4n1), and the per-launch
# counters of FlashAttention-4's d = 128 forward / backward next to this build's on the same batch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r10_smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r10_bench.json 2> gpurun_out/r10_bench.err
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__block_size,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__inst_executed_pipe_fmaheavy.sum,smsp__inst_executed_pipe_fmalite.sum,smsp__inst_executed_pipe_xu.sum,smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_tmem.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"cutlass|[Ff]lash|fmha|Sm100|attn_" -c 8 --csv --log-file gpurun_out/r10_fa4_s4n1.csv python tools/comparators.py --config S4n1 --impls fa4,ours --reps 1 > gpurun_out/r10_fa4.log 2>&1
ls -la gpurun_out
