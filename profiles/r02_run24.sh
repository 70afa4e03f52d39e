# Round 2 (session 2), GPU call 24: setmaxnreg in the forward, second try -- the TMA / MMA warpgroup
# now executes ONE setmaxnreg.dec at one program point (run 23's per-role placement hung: the four
# warps of a warpgroup must meet on the same instruction). Guarded: a 90 s smoke first.
mkdir -p gpurun_out
export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_maxnreg.so
timeout 90 python -m pytest tests/test_gpu_attention.py -q -x -k "test_fwd_bf16_local_ragged and 8-2-128" > gpurun_out/r24_smoke.log 2>&1
rc=$?
echo "exit $rc" >> gpurun_out/r24_smoke.log
if [ $rc -ne 0 ]; then echo "maxnreg smoke failed"; exit 0; fi
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r24_parity.log 2>&1
echo "exit $?" >> gpurun_out/r24_parity.log
unset SKR_LIB_PATH
VARIANTS="maxnreg" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1200 bash profiles/ab.sh > gpurun_out/r24_ab.log 2>&1
ls gpurun_out | grep r24
