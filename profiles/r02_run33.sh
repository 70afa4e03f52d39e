# Round 2 (session 3), GPU call 33: full-size parity of the alternative CP exchanges (C3n2 sampled and
# the whole 8269-token Qwen-7B sequence at N = 8 through the ring (row f4) and the fused peer exchange
# (row f3)); the CTA-pair forward variant (libskrull_fwd2sm.so) against the production forward on S4n1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k "ring or fused" > gpurun_out/r33_fullsize_exchanges.log 2>&1
echo "exit $?" >> gpurun_out/r33_fullsize_exchanges.log
VARIANTS="fwd2sm" CFGS="S4n1" STEPS=5 timeout 1200 bash profiles/ab.sh > gpurun_out/r33_ab_fwd2sm.log 2>&1
ls gpurun_out | grep r33
