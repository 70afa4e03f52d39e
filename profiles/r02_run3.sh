# Round 2, GPU call 3: where the d = 128 forward's time goes (event trace + phase accounting of
# block (0, 0) on one 8K / 16K sequence), compute-sanitizer on toy C1, f1 emulation with the
# exchange charged.
mkdir -p gpurun_out
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_evtrace.so timeout 300 python profiles/trace_fwd.py 128 0 > gpurun_out/r3_trace_fwd128.log 2>&1
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_evtrace.so timeout 300 python profiles/trace_fwd.py 128 3000 > gpurun_out/r3_trace_fwd128_late.log 2>&1
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_phase.so timeout 300 python profiles/phase_fwd.py 128 16384 > gpurun_out/r3_phase_fwd128.log 2>&1
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_phase.so timeout 300 python profiles/phase_fwd.py 64 16384 > gpurun_out/r3_phase_fwd64.log 2>&1
for tool in memcheck initcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python profiles/sanitize_c1.py > gpurun_out/r3_sanitizer_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/r3_sanitizer_$tool.log
done
for c in C5n8 C4; do timeout 1200 python tools/emulate_cp.py --config $c >> gpurun_out/r3_emulate_cp.jsonl 2>> gpurun_out/r3_emulate_cp.err; done
ls -la gpurun_out
