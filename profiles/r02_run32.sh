# Round 2 (session 3), GPU call 32: evidence of the final build (forward MMA thread issues PV_A(j-1)
# before the K(j) wait) -- smoke, the whole GPU suite, compute-sanitizer on toy C1, bench lines, the
# launch list and full captures of both kernels of the default command, the reference arm.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r32_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r32_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r32_gpu_tests.log
for t in memcheck racecheck initcheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python profiles/sanitize_c1.py > gpurun_out/r32_sanitizer_$t.log 2>&1
  echo "exit $?" >> gpurun_out/r32_sanitizer_$t.log
done
timeout 900 python bench.py > gpurun_out/r32_bench_s4n1.json 2> gpurun_out/r32_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r32_bench_c2.json 2> gpurun_out/r32_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r32_bench_c5n1.json 2> gpurun_out/r32_bench_c5n1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r32_bench_reference.json 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out/r02e
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e/launches.csv $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/r02e/prof_bwd $CMD > gpurun_out/r32_prof_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/r02e/prof_fwd $CMD > gpurun_out/r32_prof_fwd.log 2>&1
ls -la gpurun_out gpurun_out/r02e | grep -E "r32|prof|launch"
