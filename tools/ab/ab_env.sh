# A/B of an environment variable ($1=NAME, A: $1=$2, B: $1=$3), 3 benches each, interleaved
for i in 1 2 3; do for v in "$2" "$3"; do
env $1=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/e_${v}_${i}.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/e_${v}_${i}.json').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms']
print('$1=$v', round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items() if a.startswith('field')})"; done; done
