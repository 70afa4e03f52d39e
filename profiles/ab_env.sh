# A/B of an environment knob on the production library: base (unset) vs each "NAME=VALUE" in ENVS
for r in 1 2; do for e in base $ENVS; do
  for c in ${CFGS:-C5n1}; do
    if [ $e = base ]; then out=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1);
    else out=$(env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1); fi
    echo "$e $c $(echo "$out" | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*' | tr '\n' ' ')"
  done
done; done
