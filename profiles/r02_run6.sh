# Round 2, GPU call 6: the one-warpgroup-per-head d = 64 forward (libskrull_wg64.so) -- parity,
# A/B on C2, cycles per launch.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_wg64.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_cp.py -q -x -p no:cacheprovider -k "64 or rollback or fuzz or c1" > gpurun_out/r6_parity_wg64.log 2>&1
echo "exit $?" >> gpurun_out/r6_parity_wg64.log
VARIANTS="wg64" CFGS="C2" STEPS=30 timeout 900 bash profiles/ab.sh > gpurun_out/r6_ab_wg64.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
for v in base wg64; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:attn_fwd --csv --log-file gpurun_out/r6_cyc_${v}_C2.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --config C2 > /dev/null 2>&1
done
ls gpurun_out | grep r6
