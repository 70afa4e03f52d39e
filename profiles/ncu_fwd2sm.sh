# one --set full capture of the 2-CTA d=128 forward (C5n1 bench launch), for the stall breakdown
SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_fwd2sm.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd2sm -s 3 -c 1 -o gpurun_out/prof_fwd2sm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config C5n1 > gpurun_out/prof_fwd2sm.log 2>&1
