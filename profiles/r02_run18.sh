# Round 2 (session 2), GPU call 18: row split + split P hand-over (libskrull_splitp.so,
# -DSKR_FWD_SPLITP=1) -- parity and A/B against the row-split production build.
mkdir -p gpurun_out
export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_splitp.so
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r18_parity_sp.log 2>&1
echo "exit $?" >> gpurun_out/r18_parity_sp.log
unset SKR_LIB_PATH
VARIANTS="splitp" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r18_ab_sp.log 2>&1
ls gpurun_out | grep r18
