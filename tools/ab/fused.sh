# gather fused into the two-tile forward (default) vs gather kernel + two-tile forward (NS2B_FWD=2)
export NS2B_PARITY_LOG=gpurun_out/parity_fused.jsonl; rm -f $NS2B_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_mlp.py tests/test_gpu_hash_encoding.py tests/test_dynamic.py -q -p no:cacheprovider > gpurun_out/par_fused.log 2>&1; echo "fused parity rc $?"; grep -E "^FAILED|passed|failed|Error" gpurun_out/par_fused.log | tail -6
for v in 3 2 3 2; do NS2B_FWD=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_f$v.json 2> gpurun_out/b_f$v.err; python -c "
import json; d=json.loads(open('gpurun_out/b_f$v.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('FWD=$v', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})" || tail -3 gpurun_out/b_f$v.err; done
