# Round 2, GPU call 7: GPU suite after row f3 step two (dK/dV reduced from the backward kernel's
# epilogue into the owners' accumulators) and the NVTX ranges; the peer paths first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_peer_ipc.py tests/test_gpu_bench_multirank.py -q -p no:cacheprovider -k "peer or fuzz or two" > gpurun_out/r7_peer_tests.log 2>&1
echo "exit $?" >> gpurun_out/r7_peer_tests.log
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r7_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r7_tests.log
tail -3 gpurun_out/r7_tests.log
