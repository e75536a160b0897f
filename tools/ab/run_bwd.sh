# parity of the current MLP kernels, 2 benches, phase profile
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py -q -x -p no:cacheprovider -k "field_forward_backward or train_steps or flat" > gpurun_out/par.log 2>&1; echo "parity rc $?"; tail -2 gpurun_out/par.log
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), {a: round(b,3) for a,b in k.items()})"; done
NS2B_NVCC_EXTRA=-DNS2B_PHASE_PROF python -m paper_2212_05231_b200.build --force > /dev/null
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu 2>/dev/null | grep PHASEPROF | tail -2
python -m paper_2212_05231_b200.build --force > /dev/null
