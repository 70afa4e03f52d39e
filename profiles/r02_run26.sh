# Round 2 (session 2), GPU call 26: forward row sums after the P hand-over (libskrull_latesum.so,
# -DSKR_FWD_LATE_SUM=1) -- parity and A/B.
mkdir -p gpurun_out
export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_latesum.so
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r26_parity.log 2>&1
echo "exit $?" >> gpurun_out/r26_parity.log
unset SKR_LIB_PATH
VARIANTS="latesum" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1200 bash profiles/ab.sh > gpurun_out/r26_ab.log 2>&1
ls gpurun_out | grep r26
