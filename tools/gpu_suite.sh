# round-2 GPU check: c2 / data-parallel parity tests (errors logged), the full GPU suite, two benches
export NS2B_PARITY_LOG=gpurun_out/parity_r02c.jsonl
rm -f $NS2B_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_c2_step.py tests/test_gpu_parallel.py -q -s -p no:cacheprovider > gpurun_out/new_tests.log 2>&1; echo "new tests rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/new_tests.log | tail -8
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "all gpu rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/gpu_all.log | tail -8
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), {a: round(b,3) for a,b in k.items()}, d['roofline']['l2_probe'])"; done
