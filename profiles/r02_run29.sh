# Round 2 (session 3), GPU call 29: the state restored from the last checkpoint (scale fold off,
# pv_done committed once when P aliases S) -- smoke, the whole GPU suite, bench lines, launch list.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r29_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r29_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r29_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r29_bench_s4n1.json 2> gpurun_out/r29_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r29_bench_c2.json 2> gpurun_out/r29_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r29_bench_c5n1.json 2> gpurun_out/r29_bench_c5n1.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r29_launches.csv $CMD > /dev/null 2>&1
ls -la gpurun_out | grep r29
