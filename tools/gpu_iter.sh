# iteration check: parity subset + c2 tests + 2 benches + the launch list (filtered to our kernels)
export NS2B_PARITY_LOG=gpurun_out/parity_cur.jsonl; rm -f $NS2B_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_mlp.py tests/test_gpu_parallel.py -q -p no:cacheprovider > gpurun_out/par.log 2>&1; echo "parity rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/par.log | tail -6
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,3), {a: round(b,3) for a,b in k.items()})"; done
if [ -n "$1" ]; then timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(march|field|composite|adam|finite|occupancy|DeviceScan|rays)' -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"; fi
