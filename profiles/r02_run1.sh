# Round 2, GPU call 1: the full -m gpu suite (new NCCL / whole-sequence / tolerance tests), the new
# default bench (S4n1), grid-order A/B (production vs libskrull_hm.so) and DRAM bytes per launch.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r1_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r1_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r1_tests.log
timeout 600 python bench.py > gpurun_out/r1_bench_s4n1.json 2> gpurun_out/r1_bench_s4n1.err
export VARIANTS=hm CFGS="S4n1 C2 C5n1"
timeout 900 bash profiles/ab.sh > gpurun_out/r1_ab_hm.log 2>&1
for v in base hm; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_hm.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:attn_ --csv \
    --log-file gpurun_out/r1_dram_${v}_s4n1.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --config S4n1 > /dev/null 2>&1
done
unset SKR_LIB_PATH
ls -la gpurun_out
