# Round 2 (session 2), GPU call 28: the whole GPU suite with the scale fold off and pv_done committed
# once (P aliasing S); bench lines of that build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r28_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r28_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r28_bench_s4n1.json 2> gpurun_out/r28_bench_s4n1.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r28_bench_c2.json 2> gpurun_out/r28_bench_c2.err
timeout 600 python bench.py --config C5n1 --no-cpu-baseline > gpurun_out/r28_bench_c5n1.json 2> gpurun_out/r28_bench_c5n1.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r28_smoke.log 2>&1
ls gpurun_out | grep r28
