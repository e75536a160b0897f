python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -1 gpurun_out/par.log
for i in 1 2; do python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2>gpurun_out/bench2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench2.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items() if k.startswith('field')})"; done
