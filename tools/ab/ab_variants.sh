# on the box: interleaved benches of prebuilt _variants/<name>.so (R rounds), then parity per variant
# usage: R=2 K="pytest -k expr" bash tools/ab/ab_variants.sh base v1 v2 ...   (K empty: no parity)
R=${R:-2}
for i in $(seq 1 $R); do for v in "$@"; do
  cp _variants/$v.so paper_2212_05231_b200/libns2b.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/v_${v}_$i.json 2>gpurun_out/v_${v}_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/v_${v}_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('$v', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})" || tail -3 gpurun_out/v_${v}_$i.err
done; done
if [ -n "$K" ]; then for v in "$@"; do
  cp _variants/$v.so paper_2212_05231_b200/libns2b.so
  echo "parity $v: $(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_c3.py -q -p no:cacheprovider -k "$K" 2>&1 | grep -E "passed|failed|FAILED|Error" | tail -4)"
done; fi
cp _variants/base.so paper_2212_05231_b200/libns2b.so
