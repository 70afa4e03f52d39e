# Round 2 (session 2), GPU call 14: one mbarrier poller per warpgroup (libskrull_poll1.so,
# -DSKR_ONE_POLLER) vs production -- parity of the variant, per-launch counters (cycles, clock,
# instructions, LSU shared wavefronts), interleaved A/B on S4n1 / C2 / C5n1.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_poll1.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r14_parity_poll1.log 2>&1
echo "exit $?" >> gpurun_out/r14_parity_poll1.log
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for v in base poll1; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_(fwd|bwd)_kernel" -c 2 --csv --log-file gpurun_out/r14_cnt_${v}_S4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_(fwd|bwd)_kernel" -c 2 --csv --log-file gpurun_out/r14_cnt_${v}_C2.csv python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
unset SKR_LIB_PATH
VARIANTS="poll1" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r14_ab_poll1.log 2>&1
ls gpurun_out | grep r14
