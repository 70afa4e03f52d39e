# Round 2 (session 2), GPU call 17: the row-split forward softmax (libskrull_rowsplit.so,
# -DSKR_FWD_ROWSPLIT=1: each warp owns 16 rows x all key columns via 16x256b TMEM loads, shuffles
# instead of the shared-memory max exchange) -- parity, counters, A/B.
mkdir -p gpurun_out
export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_rowsplit.so
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r17_parity_rs.log 2>&1
echo "exit $?" >> gpurun_out/r17_parity_rs.log
timeout 900 python -m pytest tests/test_gpu_cp.py -q -x -k "fuzz or ring or c1" > gpurun_out/r17_parity_rs_cp.log 2>&1
echo "exit $?" >> gpurun_out/r17_parity_rs_cp.log
unset SKR_LIB_PATH
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
for v in base rowsplit; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_fwd_kernel" -c 1 --csv --log-file gpurun_out/r17_cnt_${v}_S4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_fwd_kernel" -c 1 --csv --log-file gpurun_out/r17_cnt_${v}_C2.csv python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
unset SKR_LIB_PATH
VARIANTS="rowsplit" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r17_ab_rs.log 2>&1
ls gpurun_out | grep r17
