# final check: full GPU suite, smoke(), the bench line (with the CPU leg) and the reference arm
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gpu_all.log 2>&1; echo "gpu suite rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/final_gpu_all.log | tail -6
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/final_bench.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), d['clocks'], {a: round(b,3) for a,b in k.items()})"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc $?"; tail -c 400 gpurun_out/final_bench_ref.json
