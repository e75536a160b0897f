# Config 3: tcgen05 second-order path vs torch double backward (loop / vectorised /
# torch.compile baselines), accuracy at 2^22 vs fp64, and the Theorem-1 MLP bench
for o in uniform rays; do timeout 900 python tools/bench_c3.py --points 22 --order $o --compile 2>gpurun_out/c3_$o.err | tail -1; done
timeout 900 python tools/bench_c3.py --points 22 --order rays --check64 2>gpurun_out/c3_64.err | tail -1
timeout 600 python -c "
import json
from paper_2212_05231_b200 import autodiff_oracle as a
rows = a.bench_second_order(64, 2, [1024, 4096, 16384, 65536])
print(a.bench_rows_to_csv(rows))
"
