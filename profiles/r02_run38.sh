# Round 2 (session 3), GPU call 38: same-box library context with the final build (tools/comparators.py):
# this library vs FlashAttention-4 (CuTe DSL), FlashAttention-2 and cuDNN SDPA on S4n1, C5n1, C2.
mkdir -p gpurun_out
timeout 900 python tools/comparators.py --config S4n1 --impls ours,fa4,fa2,cudnn --reps 2 > gpurun_out/r38_comparators.jsonl 2> gpurun_out/r38_comparators.err
timeout 600 python tools/comparators.py --config C5n1 --impls ours,fa4,fa2,cudnn --reps 3 >> gpurun_out/r38_comparators.jsonl 2>> gpurun_out/r38_comparators.err
timeout 600 python tools/comparators.py --config C2 --impls ours,fa4,fa2,cudnn --reps 3 >> gpurun_out/r38_comparators.jsonl 2>> gpurun_out/r38_comparators.err
ls gpurun_out | grep r38
