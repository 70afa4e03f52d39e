# Round 2 (session 2), GPU call 27: (1) synccheck of the build that commits pv_done only after the
# last PV when P aliases S; (2) which change moved the C3n2 full-size dV error (run 25 failure): the
# sampled C3n2 parity with the libraries of dd7a67b (pre scale-fold), 63e3888 (fold), ad2ccb5 (ring,
# k_len clamp) and the current build.
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool synccheck python profiles/sanitize_c1.py > gpurun_out/r27_synccheck.log 2>&1
echo "exit $?" >> gpurun_out/r27_synccheck.log
for v in cur vdd7a67b v63e3888 vad2ccb5; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  echo "== $v" >> gpurun_out/r27_c3n2.log
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "C3n2" 2>&1 | grep -E "passed|failed|err .* >|bf16 d[kqv] |bf16 o " >> gpurun_out/r27_c3n2.log
done
ls gpurun_out | grep r27
