# A/B: current tree vs tools/_ab_patch (rebuilt on the box); 3 bench runs each
run3() { for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']; print('$1', round(d['ms_per_step'],3), round(k['field_mlp_forward'],3), round(k['field_mlp_backward'],3), round(k['field_gather'],3), round(k['field_scatter'],3))"; done; }
run3 A
git apply "$1" && python -m paper_2212_05231_b200.build > /dev/null && run3 B
if [ -n "$2" ]; then python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; fi
