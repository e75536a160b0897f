"""tcgen05 MMA issue-rate probe for the MLP kernels' GEMM shapes (run on the GPU)."""
import torch

from paper_2212_05231_b200 import _lib

names = {0: "M128 N64 K/MN", 1: "M64 N16 MN/MN", 2: "M64 N64 MN/MN", 3: "M128 N16 K/K", 4: "M64 N8 MN/MN",
         5: "M128 N64 K/K"}
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for shape in range(6):
    for nacc in (1, 2, 4):
        row = []
        for iters in (1, 3, 12, 48, 192):
            vals = []
            for _ in range(3):
                _lib.call("ns2b_bench_umma", shape, iters, nacc, _lib.ptr(out), _lib.stream_ptr())
                torch.cuda.synchronize()
                vals.append(int(out.item()))
            row.append(f"{iters}:{min(vals)}")
        print(f"{names[shape]:16s} nacc={nacc}  cycles " + "  ".join(row))
