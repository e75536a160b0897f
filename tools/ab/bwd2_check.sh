# bwd2 bring-up: one field parity test under a timeout, then A/B (NS2B_BWD=1 vs default), then parity
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "field_forward_backward and c1" 2>&1 | tail -3
rc=$?
for i in 1 2; do for v in 1 2; do
  NS2B_BWD=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bw_${v}_$i.json 2>gpurun_out/bw_${v}_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/bw_${v}_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('BWD=$v', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})" || tail -3 gpurun_out/bw_${v}_$i.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_c3.py tests/test_gpu_mlp.py tests/test_dynamic.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|FAILED|Error" | tail -8
