# Round 2 (session 3), GPU call 31: d = 128 forward variants -- a 5-unit K/V ring (units5), the MMA
# thread issuing PV_A(j-1) before waiting for K(j) (pvfirst), both -- parity of each on the attention
# suite, then interleaved A/B against the production library on S4n1 and C5n1.
mkdir -p gpurun_out
for v in units5 pvfirst both; do
  SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "not fuzz" > gpurun_out/r31_parity_$v.log 2>&1
  echo "exit $?" >> gpurun_out/r31_parity_$v.log
done
VARIANTS="units5 pvfirst both" CFGS="S4n1 C5n1" STEPS=5 timeout 2400 bash profiles/ab.sh > gpurun_out/r31_ab.log 2>&1
ls gpurun_out | grep r31
