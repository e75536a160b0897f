# A/B of a compile flag ($1): 2 benches each (A = default build, B = -D$1), then parity of B
run() { for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_$1_$i.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_$1_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('$1', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})"; done; }
run A
NS2B_NVCC_EXTRA="-D$1" python -m paper_2212_05231_b200.build --force > /dev/null
run B
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py -q -x -p no:cacheprovider -k "field_forward_backward or train_steps or flat" 2>&1 | tail -1
python -m paper_2212_05231_b200.build --force > /dev/null
