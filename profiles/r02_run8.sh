# Round 2, GPU call 8: the profiling recipe on the default bench command (S4n1): launch list, one
# `ncu --set full` capture of each attention kernel; final bench lines (default, C2, C5n1, the
# reference arm) and smoke.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/prof_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/prof_fwd.log 2>&1
timeout 900 python bench.py > gpurun_out/r8_bench_default.json 2> gpurun_out/r8_bench_default.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r8_bench_c2.json 2> gpurun_out/r8_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r8_bench_c5n1.json 2> gpurun_out/r8_bench_c5n1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r8_bench_reference.json 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r8_smoke.log 2>&1
ls -la gpurun_out | grep -E "prof_|launches|r8_"
# exp2 polynomial share under the power cap (env knobs, same library): interleaved A/B
for r in 1 2; do
  for fp in 1 0; do
    echo "fwd_poly=$fp S4n1 $(SKR_FWD_POLY=$fp timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r8_ab_poly.log
  done
  for fp in 2 1 0; do
    echo "fwd_poly=$fp C2 $(SKR_FWD_POLY=$fp timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r8_ab_poly.log
  done
done
