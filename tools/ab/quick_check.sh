# quick GPU check of the working tree: targeted parity tests ($1 = pytest -k expr), then 2 benches
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_c3.py tests/test_gpu_mlp.py tests/test_gpu_parallel.py -q -p no:cacheprovider -k "$1" 2>&1 | grep -E "passed|failed|FAILED|Error" | tail -6
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/q_$i.json 2>gpurun_out/q_$i.err
python -c "
import json; d=json.loads(open('gpurun_out/q_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), {a: round(b,3) for a,b in k.items()})" || tail -3 gpurun_out/q_$i.err; done
