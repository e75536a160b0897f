# Full GPU test suite, then two 10-step bench runs (kernel times).
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']; print('run', round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,3), round(k['field_mlp_forward'],3), round(k['field_mlp_backward'],3), round(k['field_gather'],3), round(k['field_scatter'],3))"; done
