# Round 2 (session 2), GPU call 23: setmaxnreg in the forward (libskrull_maxnreg.so: 20 warps, the
# TMA / MMA warpgroup at 56 registers, the softmax warps at 112 instead of 96) -- parity, A/B, counters.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_maxnreg.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/r23_parity.log 2>&1
echo "exit $?" >> gpurun_out/r23_parity.log
VARIANTS="maxnreg" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r23_ab.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for v in base maxnreg; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_fwd_kernel" -c 1 --csv --log-file gpurun_out/r23_cnt_${v}_S4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_fwd_kernel" -c 1 --csv --log-file gpurun_out/r23_cnt_${v}_C2.csv python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out | grep r23
