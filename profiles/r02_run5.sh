# Round 2, GPU call 5: is the step power-bound? Cycles vs time per attention launch (ncu, clocks not
# controlled) for the production library and the one-warpgroup forward, plus power draw under load.
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum
for v in base wg1; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  for c in S4n1 C5n1; do
    timeout 600 ncu --metrics $M --clock-control none -k regex:attn_ --csv --log-file gpurun_out/r5_cyc_${v}_${c}.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --config $c > /dev/null 2>&1
  done
done
unset SKR_LIB_PATH
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > gpurun_out/r5_power_base.csv &
P=$!
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r5_bench_base.json 2>&1
kill $P
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > gpurun_out/r5_power_wg1.csv &
P=$!
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_wg1.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r5_bench_wg1.json 2>&1
kill $P
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 99 python profiles/sanitize_c1.py > gpurun_out/r5_sanitizer_synccheck.log 2>&1
echo "exit $?" >> gpurun_out/r5_sanitizer_synccheck.log
ls gpurun_out | grep r5
