"""tcgen05 grouped GEMM throughput at prefill shapes (TFLOP/s vs MEASURED_PEAKS)."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200 import kernels as K_  # noqa: E402

dev = torch.device("cuda")
pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
res = {}
for name, T, k, E, d, I in (("mixtral_prefill2k", 2048, 2, 8, 4096, 14336), ("qwen_prefill512", 512, 4, 60, 2048, 1408),
                            ("dseek_batch256", 256, 6, 64, 2048, 1408), ("dense_8k", 8192, 1, 1, 4096, 4096),
                            ("dseek_decode64", 64, 3, 64, 2048, 1408), ("mixtral_decode8", 8, 2, 8, 4096, 14336)):
    g = torch.Generator(device=dev).manual_seed(0)
    P = T * k
    rows13 = 2 * I
    W = (torch.randn(E, rows13 * d + d * I, device=dev, generator=g) * 0.02).bfloat16()
    idx = torch.stack([torch.randperm(E, device=dev, generator=g)[:k] for _ in range(T)]).int() if E > 1 else \
        torch.zeros(T, 1, dtype=torch.int32, device=dev)
    perm = K_.permute(idx, torch.full((T,), k, dtype=torch.int32, device=dev), E)
    X = torch.randn(P, d, device=dev).bfloat16()
    U = torch.empty(P, I, device=dev, dtype=torch.bfloat16)
    Y = torch.empty(P, d, device=dev)
    mt = (P + 127) // 128 + min(E, P)

    def run():
        K_.grouped_gemm(X, d, W.data_ptr(), W.shape[1] * 2, E, rows13, offsets=perm["offsets"], active=perm["active"],
                        max_tiles=mt * (rows13 // 128), epi=K_.GG_SWIGLU_BF16, out_bf16=U, ldo=I)
        K_.grouped_gemm(U, I, W.data_ptr() + rows13 * d * 2, W.shape[1] * 2, E, d, offsets=perm["offsets"],
                        active=perm["active"], max_tiles=mt * (d // 128), epi=K_.GG_STORE_F32, out_f32=Y, ldo=d,
                        row_to_pair=perm["sorted_pairs"])
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 2.0 * P * (rows13 * d + d * I)
    tf = flops / (ms / 1e3) / 1e12
    res[name] = dict(ms=round(ms, 3), TFLOPs=round(tf, 1), frac_burst=round(tf / pk["bf16_tflops"], 3),
                     frac_sustained=round(tf / pk["bf16_tflops_sustained"], 3), GFLOP=round(flops / 1e9, 1))
    # weight bytes of the experts that received rows (the decode-batch bound: a weight stream)
    n_act = int(perm["active"][0].item())
    wb = n_act * (rows13 * d + d * I) * 2
    res[name].update(weight_GBs=round(wb / ms / 1e6, 1),
                     weight_frac_hbm=round(wb / ms / 1e6 / pk["hbm_gbs"], 3))
    del W, X, U, Y
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
