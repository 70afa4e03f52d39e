# Round 2 (session 3), GPU call 35: evidence of the final build (tcgen05 fence after the forward's
# K(j) wait) -- smoke, the whole GPU suite (incl. the full-size ring / fused exchange cases), bench
# lines, the launch list of the default command.
mkdir -p gpurun_out/r02f
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r35_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r35_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r35_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r35_bench_s4n1.json 2> gpurun_out/r35_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r35_bench_c2.json 2> gpurun_out/r35_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r35_bench_c5n1.json 2> gpurun_out/r35_bench_c5n1.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f/launches.csv $CMD > /dev/null 2>&1
ls -la gpurun_out | grep r35
