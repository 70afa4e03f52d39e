set -x
for CFG in C2 C5n1; do
  D=gpurun_out/ncu_$CFG; mkdir -p $D
  CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config $CFG"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $CMD > $D/launches.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o $D/prof_bwd $CMD > $D/prof_bwd.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o $D/prof_fwd $CMD > $D/prof_fwd.log 2>&1
done
ls -la gpurun_out/ncu_*
