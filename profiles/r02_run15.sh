# Round 2 (session 2), GPU call 15: the backward with scale * P folded into the exponent
# (libskrull_fold.so, -DSKR_BWD_SCALE_FOLD=1) -- parity, counters, A/B; the bench's multi-rank flow
# on the default workload at N = 2 (S4n2, two ranks sharing the GPU).
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_fold.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r15_parity_fold.log 2>&1
echo "exit $?" >> gpurun_out/r15_parity_fold.log
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_fold.so timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "whole" > gpurun_out/r15_parity_fold_full.log 2>&1
echo "exit $?" >> gpurun_out/r15_parity_fold_full.log
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for v in base fold; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_bwd_kernel" -c 1 --csv --log-file gpurun_out/r15_cnt_${v}_S4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_bwd_kernel" -c 1 --csv --log-file gpurun_out/r15_cnt_${v}_C2.csv python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
unset SKR_LIB_PATH
VARIANTS="fold" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r15_ab_fold.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_multirank.py -q -x > gpurun_out/r15_multirank.log 2>&1
echo "exit $?" >> gpurun_out/r15_multirank.log
ls gpurun_out | grep r15
