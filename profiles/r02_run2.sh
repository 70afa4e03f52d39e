# Round 2, GPU call 2: backward step-order variants (parity + A/B + DRAM), same-box library
# comparators (FA2 / FA4 / cuDNN), and the GPU suite on the head-major production library.
mkdir -p gpurun_out
for v in bo1 bo2; do
  SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider -k "bwd" > gpurun_out/r2_parity_$v.log 2>&1
  echo "exit $?" >> gpurun_out/r2_parity_$v.log
done
VARIANTS="bo1 bo2" CFGS="S4n1 C5n1 C2" STEPS=5 timeout 1200 bash profiles/ab.sh > gpurun_out/r2_ab_bwd_order.log 2>&1
for v in base bo1 bo2; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:attn_ --csv \
    --log-file gpurun_out/r2_dram_${v}_s4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config S4n1 > /dev/null 2>&1
done
unset SKR_LIB_PATH
for c in S4n1 C5n1 C2; do timeout 900 python tools/comparators.py --config $c >> gpurun_out/r2_comparators.jsonl 2>> gpurun_out/r2_comparators.err; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r2_tests.log
ls -la gpurun_out
