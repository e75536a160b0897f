# on the box: phase profiles (NS2B_PHASE_PROF builds) of prebuilt _variants/<name>.so
for v in "$@"; do cp _variants/$v.so paper_2212_05231_b200/libns2b.so
  echo "== $v"; timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu 2>/dev/null | grep PHASEPROF | tail -2; done
cp _variants/base.so paper_2212_05231_b200/libns2b.so
