# Round 2 (session 2), GPU call 16: row f4's ring CP (loopback over N = 1-4 ranks, 1-rank NCCL
# send / recv) and the k_len-clamped attention kernels -- the GPU suite parts they touch, then an
# S4n1 bench to check the production path did not move.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_nccl.py tests/test_gpu_cp.py tests/test_gpu_fwd2sm.py -q -x > gpurun_out/r16_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r16_tests.log
timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r16_bench.json 2> gpurun_out/r16_bench.err
ls gpurun_out | grep r16
