# Round 2, GPU call 7: full GPU suite after row f3 step two (dK/dV reduced from the backward
# kernel's epilogue into the owners' accumulators) and the NVTX ranges.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r7_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r7_tests.log
SKR_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --config C2 --exchange peer > gpurun_out/r7_bench_peer2.log 2>&1
tail -3 gpurun_out/r7_tests.log
