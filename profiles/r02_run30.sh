# Round 2 (session 3), GPU call 30: the GPU suite with R34'' on the full-size gradient checks
# (tests/attn_harness.operand_rounding_dev), smoke, and ncu --set full of both attention kernels of
# the default command (the scale fold is off again since r02c's capture).
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r30_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r30_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r30_gpu_tests.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/r30_prof_bwd $CMD > gpurun_out/r30_prof_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/r30_prof_fwd $CMD > gpurun_out/r30_prof_fwd.log 2>&1
ls -la gpurun_out | grep r30
