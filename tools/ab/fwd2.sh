# two-tiles-in-flight forward (default) vs the one-tile forward (NS2B_FWD=1): parity + benches
export NS2B_PARITY_LOG=gpurun_out/parity_fwd2.jsonl; rm -f $NS2B_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_step.py tests/test_gpu_mlp.py -q -p no:cacheprovider -k "field_forward_backward or train_steps or flat or chained or mlp" > gpurun_out/par_fwd2.log 2>&1; echo "fwd2 parity rc $?"; grep -E "^FAILED|passed|failed|Error" gpurun_out/par_fwd2.log | tail -4
for v in 0 1 0 1; do NS2B_FWD=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_fwd$v.json 2> gpurun_out/b_fwd$v.err; python -c "
import json; d=json.loads(open('gpurun_out/b_fwd$v.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('FWD=$v', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})" || tail -3 gpurun_out/b_fwd$v.err; done
