# Round 2 (session 2), GPU call 25: evidence of the final production build (row-split forward, spin
# MMA waits, query-banded + scale-folded backward, ring CP) -- smoke, the whole GPU suite,
# compute-sanitizer on toy C1 (incl. banded lists and the ring), bench lines, the profiling recipe
# on the default command, same-box library context.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r25_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r25_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r25_gpu_tests.log
for t in memcheck racecheck initcheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python profiles/sanitize_c1.py > gpurun_out/r25_sanitizer_$t.log 2>&1
  echo "exit $?" >> gpurun_out/r25_sanitizer_$t.log
done
timeout 900 python bench.py > gpurun_out/r25_bench_s4n1.json 2> gpurun_out/r25_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r25_bench_c2.json 2> gpurun_out/r25_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r25_bench_c5n1.json 2> gpurun_out/r25_bench_c5n1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r25_bench_reference.json 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r25_launches.csv $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/r25_prof_bwd $CMD > gpurun_out/r25_prof_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/r25_prof_fwd $CMD > gpurun_out/r25_prof_fwd.log 2>&1
timeout 900 python tools/comparators.py --config S4n1 --impls ours,fa4,fa2 --reps 2 > gpurun_out/r25_comparators_s4n1.jsonl 2> gpurun_out/r25_comparators.err
timeout 600 python tools/comparators.py --config C2 --impls ours,fa4 --reps 3 > gpurun_out/r25_comparators_c2.jsonl 2>> gpurun_out/r25_comparators.err
ls -la gpurun_out | grep r25
