# A/B: libskrull.so (A) vs libskrull_alt.so (B), interleaved, same box
for r in 1 2; do
for v in A B; do
  if [ $v = B ]; then export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_alt.so; else unset SKR_LIB_PATH; fi
  for c in ${CFGS:-C2 C5n1}; do echo "$v $c $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*' | tr '\n' ' ')"; done
done; done
