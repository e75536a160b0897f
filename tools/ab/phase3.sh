NS2B_NVCC_EXTRA=-DNS2B_PHASE_PROF python -m paper_2212_05231_b200.build --force > /dev/null
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu 2>/dev/null | grep PHASEPROF | tail -2
python -m paper_2212_05231_b200.build --force > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "field_forward_backward" 2>&1 | tail -2
NS2B_FWD=3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('FWD=3', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})"
