# Round 2, GPU call 4: the one-warpgroup-per-head d = 128 forward (libskrull_wg1.so): parity,
# interleaved A/B against production, phase accounting.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_wg1.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_cp.py -q -x -p no:cacheprovider -k "128 or cp_mixed or fuzz" > gpurun_out/r4_parity_wg1.log 2>&1
echo "exit $?" >> gpurun_out/r4_parity_wg1.log
SKR_FWD_WG=1 SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_phase_wg1.so timeout 300 python profiles/phase_fwd.py 128 16384 > gpurun_out/r4_phase_fwd128_wg1.log 2>&1
VARIANTS="wg1" CFGS="S4n1 C5n1" STEPS=5 timeout 1200 bash profiles/ab.sh > gpurun_out/r4_ab_wg1.log 2>&1
for v in base wg1; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 python profiles/long_seq.py 128 > gpurun_out/r4_longseq_$v.log 2>&1
done
ls -la gpurun_out | tail -5
