# Round 2 (session 2), GPU call 22: packed-pair polynomial exponentials in the forward (production,
# SKR_FWD_PACKED_POLY=1) vs scalar (libskrull_nopack.so), at the default shares and at 2/8 for d = 128.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r22_parity.log 2>&1
echo "exit $?" >> gpurun_out/r22_parity.log
VARIANTS="nopack" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r22_ab.log 2>&1
for r in 1 2; do
  for v in base nopack; do
    if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
    echo "$v poly2 S4n1 $(SKR_FWD_POLY=2 timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r22_poly2.log
  done
done
ls gpurun_out | grep r22
