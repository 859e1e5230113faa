"""One launch per case of the persistent grouped GEMM for an ncu --set full
capture: dense 8192x4096x4096 (tensor-bound) and the C4 batch-64 expert
gate-up (weight stream).  python scripts/prof_gemm.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200 import kernels as K_  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
# dense 8k: M=8192, N=4096, K=4096
A = torch.randn(8192, 4096, device=dev, generator=g).bfloat16()
B = torch.randn(4096, 4096, device=dev, generator=g).bfloat16()
out = torch.empty(8192, 4096, device=dev)
K_.grouped_gemm(A, 4096, B.data_ptr(), B.numel() * 2, 1, 4096, max_tiles=64 * 32, dense_rows=8192, dense_experts=1,
                epi=K_.GG_STORE_F32, out_f32=out, ldo=4096)
# C4 decode batch 64, k=3: routed gate-up (2I = 2816 rows of d = 2048) over 64 experts
T, k, E, d, I = 64, 3, 64, 2048, 1408
W = (torch.randn(E, 2 * I * d + d * I, device=dev, generator=g) * 0.02).bfloat16()
idx = torch.stack([torch.randperm(E, device=dev, generator=g)[:k] for _ in range(T)]).int()
perm = K_.permute(idx, torch.full((T,), k, dtype=torch.int32, device=dev), E)
X = torch.randn(T * k, d, device=dev).bfloat16()
U = torch.empty(T * k, I, device=dev, dtype=torch.bfloat16)
mt = (T * k + 127) // 128 + min(E, T * k)
K_.grouped_gemm(X, d, W.data_ptr(), W.shape[1] * 2, E, 2 * I, offsets=perm["offsets"], active=perm["active"],
                max_tiles=mt * (2 * I // 128), epi=K_.GG_SWIGLU_BF16, out_bf16=U, ldo=I)
torch.cuda.synchronize()
print("ok")
