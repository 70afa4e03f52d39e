for p in 0 1 2 3; do echo "POLY=$p"; SKR_FWD_POLY=$p timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"fwd_ms[^,]*'; done
SKR_FWD_POLY=2 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config C5n1 2>&1 | grep -o '"value[^,]*\|"fwd_ms[^,]*\|"bwd_ms[^,]*'
