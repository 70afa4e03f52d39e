# A/B of single long sequences (profiles/long_seq.py): production library vs libskrull_<v>.so, interleaved
for r in 1 2; do for v in base ${VARIANTS:-alt}; do
  if [ $v = base ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/paper_2505_19609_b200/libskrull_$v.so; fi
  timeout 300 python profiles/long_seq.py ${D:-128} 2>&1 | sed "s/^/$v /"
done; done
