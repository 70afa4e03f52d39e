# Round 2 (session 3), GPU call 41: how much the lone-head CTAs of odd GQA groups cost the d = 64 forward.
mkdir -p gpurun_out
timeout 600 python profiles/lone_head.py > gpurun_out/r41_lone_head.log 2>&1
ls gpurun_out | grep r41
