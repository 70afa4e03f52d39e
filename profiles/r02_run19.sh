# Round 2 (session 2), GPU call 19: exp2 polynomial share re-swept after the forward row split
# (SKR_FWD_POLY, interleaved), and a source-level full capture of the new d = 128 forward.
mkdir -p gpurun_out
for r in 1 2; do
  for fp in 1 2 0; do
    echo "fwd_poly=$fp S4n1 $(SKR_FWD_POLY=$fp timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r19_poly.log
  done
  for fp in 2 3 1; do
    echo "fwd_poly=$fp C2 $(SKR_FWD_POLY=$fp timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')" >> gpurun_out/r19_poly.log
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -c 1 -o gpurun_out/r19_prof_fwd python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r19_prof_fwd.log 2>&1
ls gpurun_out | grep r19
