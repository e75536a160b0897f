# A/B/C...: current tree, then each patch applied alone (rebuilt on the box); 3 bench runs each.
# usage: bash tools/_abn.sh p1.patch [p2.patch ...]   (NS2B_AB_PARITY=1: parity test per patch)
run3() { for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']; print('$1', round(d['ms_per_step'],3), round(k['field_mlp_forward'],3), round(k['field_mlp_backward'],3), round(k['field_gather'],3), round(k['field_scatter'],3), round(k['composite'],3), round(k['march_count_scan'],3), round(k['march_fill'],3))"; done; }
run3 base
for p in "$@"; do
  git apply "$p" && python -m paper_2212_05231_b200.build > /dev/null && run3 "$(basename $p .patch)"
  if [ -n "$NS2B_AB_PARITY" ]; then python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; fi
  git apply -R "$p"
done
python -m paper_2212_05231_b200.build > /dev/null
