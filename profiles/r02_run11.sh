# Round 2 (session 2), GPU call 11: query-banded backward work items -- parity, then S4n1 A/B of the
# band height (0 = round-1 whole key tiles) and the backward's DRAM bytes per launch.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/r11_tests_attn.log 2>&1
echo "attn tests exit $?" >> gpurun_out/r11_tests_attn.log
for r in 1 2; do
  for b in 0 8192 4096 16384; do
    echo "band=$b $(timeout 300 python bench.py --bwd-band $b --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r11_ab_band.log
  done
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for b in 0 8192 4096; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_bwd_kernel|band_kv" -c 3 --csv --log-file gpurun_out/r11_dram_band$b.csv python bench.py --bwd-band $b --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r11_tests_full.log 2>&1
echo "fullsize tests exit $?" >> gpurun_out/r11_tests_full.log
ls gpurun_out
