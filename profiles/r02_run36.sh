# Round 2 (session 3), GPU call 36: d = 64 forward MMA issue order per head ([S_s(j), PV_s(j-1)] for
# s = A, B instead of [S_A S_B][PV_A PV_B]; libskrull_order64.so) -- attention parity, then
# interleaved A/B on C2 (configs[1]).
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_order64.so timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "not fuzz" > gpurun_out/r36_parity_order64.log 2>&1
echo "exit $?" >> gpurun_out/r36_parity_order64.log
VARIANTS="order64" CFGS="C2" STEPS=10 timeout 1200 bash profiles/ab.sh > gpurun_out/r36_ab_order64.log 2>&1
VARIANTS="order64" CFGS="C2" STEPS=10 timeout 1200 bash profiles/ab.sh >> gpurun_out/r36_ab_order64.log 2>&1
ls gpurun_out | grep r36
