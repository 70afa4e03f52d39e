# Round 2 (session 3), GPU call 40: d = 128 forward with S split into N = 64 halves (P in S's second
# half, keys [0, 64) of S(j+1) issued once the softmax has loaded S(j); libskrull_ssplit.so):
# attention parity (guarded), then interleaved A/B on S4n1 and C5n1.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_ssplit.so timeout 300 python -m pytest tests/test_gpu_attention.py -q -x -k "not fuzz" > gpurun_out/r40_parity_ssplit.log 2>&1
rc=$?
echo "exit $rc" >> gpurun_out/r40_parity_ssplit.log
if [ $rc = 0 ]; then
  SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_ssplit.so timeout 600 python -m pytest tests/test_gpu_cp.py -q -x -k "peer or ring or nccl or fuzz" > gpurun_out/r40_parity_ssplit_cp.log 2>&1
  echo "exit $?" >> gpurun_out/r40_parity_ssplit_cp.log
  VARIANTS="ssplit" CFGS="S4n1 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r40_ab_ssplit.log 2>&1
fi
ls gpurun_out | grep r40
