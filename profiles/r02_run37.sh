# Round 2 (session 3), GPU call 37: the whole GPU suite with the lazily evaluated R34'' allowance
# (final test code), and the smoke.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r37_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r37_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r37_gpu_tests.log
ls gpurun_out | grep r37
