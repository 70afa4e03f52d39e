# Round 2 (session 2), GPU call 13: evidence of the banded-backward build -- full GPU suite, smoke,
# compute-sanitizer (toy C1 incl. banded lists), bench lines (default S4n1, C2, C5n1, reference
# arm), the profiling recipe on the default command (launch list + full captures).
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r13_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r13_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r13_gpu_tests.log
for t in memcheck racecheck initcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python profiles/sanitize_c1.py > gpurun_out/r13_sanitizer_$t.log 2>&1
  echo "exit $?" >> gpurun_out/r13_sanitizer_$t.log
done
timeout 900 python bench.py > gpurun_out/r13_bench_s4n1.json 2> gpurun_out/r13_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r13_bench_c2.json 2> gpurun_out/r13_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r13_bench_c5n1.json 2> gpurun_out/r13_bench_c5n1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r13_bench_reference.json 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r13_launches.csv $CMD > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/r13_prof_bwd $CMD > gpurun_out/r13_prof_bwd.log 2>&1
ls -la gpurun_out | grep r13
