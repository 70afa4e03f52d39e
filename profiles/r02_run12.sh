# Round 2 (session 2), GPU call 12: banded backward with one CTA per work item for the band
# zero / cast; S4n1 A/B (band 0 / 8192, forward with suspend-hinted S waits); forward counters and a
# source-level full capture of the d = 128 forward.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q -k "band or distributed" > gpurun_out/r12_tests_attn.log 2>&1
echo "exit $?" >> gpurun_out/r12_tests_attn.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:"band_kv|attn_bwd_kernel|attn_fwd_kernel" -c 4 --csv --log-file gpurun_out/r12_band8192.csv python bench.py --bwd-band 8192 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_sleep.so timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_fwd_kernel" -c 1 --csv --log-file gpurun_out/r12_fwd_sleep.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for r in 1 2; do
  for v in b0 b8192 sleep; do
    if [ $v = sleep ]; then export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_sleep.so; B=8192; else unset SKR_LIB_PATH; B=${v#b}; fi
    echo "$v $(timeout 300 python bench.py --bwd-band $B --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r12_ab.log
  done
done
unset SKR_LIB_PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -c 1 -o gpurun_out/r12_prof_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r12_prof_fwd.log 2>&1
ls -la gpurun_out
