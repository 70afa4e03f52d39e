# Round 2 (session 2), GPU call 20: the MMA-issuing thread's waits as a plain try_wait spin
# (libskrull_spin.so, -DSKR_MMA_SPIN) instead of the suspend-hinted wait -- A/B and counters.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_spin.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -k "128 or 64" > gpurun_out/r20_parity_spin.log 2>&1
echo "exit $?" >> gpurun_out/r20_parity_spin.log
VARIANTS="spin" CFGS="S4n1 C2 C5n1" STEPS=5 timeout 1800 bash profiles/ab.sh > gpurun_out/r20_ab_spin.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for v in base spin; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_(fwd|bwd)_kernel" -c 2 --csv --log-file gpurun_out/r20_cnt_${v}_S4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out | grep r20
