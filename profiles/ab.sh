# A/B timing: production libskrull.so (A) vs experiment builds libskrull_<v>.so (SKR_VARIANT=<v>,
# paper_2505_19609_b200/build.py), interleaved twice on the same box.
#   VARIANTS="nolds" CFGS="C2 C5n1" bash profiles/ab.sh
for r in 1 2; do
for v in base ${VARIANTS:-alt}; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  for c in ${CFGS:-C2 C5n1}; do echo "$v $c $(timeout 300 python bench.py --steps ${STEPS:-10} --warmup ${WARM:-3} --no-cpu-baseline --no-e2e --config $c 2>&1 | grep -o '"value[^,]*\|fwd_ms[^,]*\|bwd_ms[^,]*\|sm_mhz[^,]*' | tr '\n' ' ')"; done
done; done
