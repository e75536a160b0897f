"""B200-native NeuS2 static training hot path (arXiv 2212.05231).

Module layout mirrors the reference package `hashsdf`:
    hash_encoding, relu_mlp, field, renderer, trainer, scene_io, _kernels
backed by the C-ABI CUDA library libns2b.so (include/ns2b.h, csrc/*.cu, sm_100a).
There is no CPU fallback: importing works anywhere, calling needs the built
library and a CUDA device.
"""

__version__ = "0.1.0"
