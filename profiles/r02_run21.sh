# Round 2 (session 2), GPU call 21: forward MMA thread on plain try_wait + the redundant pv_done wait
# skipped when P aliases S (production build) vs the previous commit (libskrull_prev.so): parity, A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_cp.py -q -x -k "not fuzz" > gpurun_out/r21_parity.log 2>&1
echo "exit $?" >> gpurun_out/r21_parity.log
VARIANTS="prev" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r21_ab.log 2>&1
ls gpurun_out | grep r21
