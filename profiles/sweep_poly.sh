# share of exponentials (per 8) on the FMA pipe: forward (SKR_FWD_POLY) and backward (SKR_BWD_POLY)
for p in ${POLYS:-0 1 2 3 4}; do for c in ${CFGS:-C2 C5n1}; do
  echo "FWD_POLY=$p $c $(SKR_FWD_POLY=$p timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1 | grep -o '"fwd_ms[^,]*')"
  echo "BWD_POLY=$p $c $(SKR_BWD_POLY=$p timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1 | grep -o '"bwd_ms[^,]*')"
done; done
