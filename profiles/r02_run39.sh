# Round 2 (session 3), GPU call 39: the whole 8269-token Qwen2.5-0.5B (d = 64) sequence at N = 8
# through the ring and fused peer exchanges (new full-size cases).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -k "qwen05" > gpurun_out/r39_fullsize_qwen05.log 2>&1
echo "exit $?" >> gpurun_out/r39_fullsize_qwen05.log
ls gpurun_out | grep r39
