"""tcgen05/TMEM/TMA grouped expert GEMM (prefill / batched path) on the GPU.

Reference: fp32 products of the same bf16 operands (the GEMM's inputs are
bf16; accumulation is f32 in TMEM), so the tolerance only covers summation
order: rel <= 1e-3 (bf16-rounded intermediates where the kernel rounds).
"""
import numpy as np
import pytest
import torch

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(cuda_ok):
    return torch.device("cuda")


@pytest.mark.parametrize("M,N,K,S", [(128, 128, 64, 1), (200, 256, 128, 2), (1000, 384, 2048, 3), (77, 128, 1408, 1)])
def test_dense_gemm(dev, M, N, K, S):
    from paper_2510_12357_b200 import kernels as K_
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    B = torch.randn(S, N, K, device=dev, generator=g).to(torch.bfloat16)
    out = torch.full((M, S * N), float("nan"), device=dev)
    tiles = S * ((M + 127) // 128) * (N // 128)
    K_.grouped_gemm(A, K, B.data_ptr(), N * K * 2, S, N, max_tiles=tiles, dense_rows=M, dense_experts=S,
                    epi=K_.GG_STORE_F32, out_f32=out, ldo=S * N, out_expert_stride=N)
    torch.cuda.synchronize()
    for e in range(S):
        want = A.float() @ B[e].float().T
        got = out[:, e * N:(e + 1) * N]
        assert rel_err(got.cpu().numpy(), want.cpu().numpy()) < 1e-3, e


@pytest.mark.parametrize("M,N,K", [(64, 2048, 2048), (8, 6144, 2048), (256, 2048, 4096), (5, 384, 1024)])
def test_dense_split_k_accumulate(dev, M, N, K):
    """Decode-batch projections (few tiles, long K): the split-K path, with
    the residual-accumulate epilogue; reruns are bit-identical (partials are
    summed in split order by the tile's last CTA)."""
    from paper_2510_12357_b200 import kernels as K_
    g = torch.Generator(device=dev).manual_seed(M * 7 + N)
    A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device=dev, generator=g).to(torch.bfloat16)
    resid = torch.randn(M, N, device=dev, generator=g)
    tiles = ((M + 127) // 128) * (N // 128)
    outs = []
    for _ in range(3):
        out = resid.clone()
        K_.grouped_gemm(A, K, B.data_ptr(), N * K * 2, 1, N, max_tiles=tiles, dense_rows=M, dense_experts=1,
                        epi=K_.GG_ACCUM_F32, out_f32=out, ldo=N)
        outs.append(out)
    torch.cuda.synchronize()
    want = resid + A.float() @ B.float().T
    assert rel_err(outs[0].cpu().numpy(), want.cpu().numpy()) < 1e-3
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("T,k,E,d,I", [(64, 2, 8, 128, 64), (300, 4, 12, 256, 128), (2048, 2, 8, 512, 256),
                                       (513, 4, 60, 2048, 1408)])
def test_grouped_expert_ffn(dev, T, k, E, d, I):
    """Routed experts end to end: gather -> gate-up (SwiGLU, bf16 U) -> down (f32, scattered to pairs)."""
    from paper_2510_12357_b200 import kernels as K_
    from paper_2510_12357_b200.weights import pack_experts
    g = torch.Generator(device=dev).manual_seed(T * 7 + E)
    w_in = (torch.rand(E, d, I, device=dev, generator=g) * 2 - 1) / d ** 0.5
    w_up = (torch.rand(E, d, I, device=dev, generator=g) * 2 - 1) / d ** 0.5
    w_out = (torch.rand(E, I, d, device=dev, generator=g) * 2 - 1) / I ** 0.5
    packed = pack_experts(w_in.bfloat16(), w_up.bfloat16(), w_out.bfloat16())  # (E, P)
    P_el = packed.shape[1]
    w13_el = 2 * I * d
    h2 = torch.randn(T, d, device=dev, generator=g)
    idx = torch.stack([torch.randperm(E, device=dev, generator=g)[:k] for _ in range(T)]).int()
    k_tok = torch.full((T,), k, dtype=torch.int32, device=dev)
    perm = K_.permute(idx, k_tok, E)
    P = T * k
    X = torch.empty(P, d, device=dev, dtype=torch.bfloat16)
    K_.gather_bf16(h2, perm["sorted_pairs"], k, P, X)
    U = torch.empty(P, I, device=dev, dtype=torch.bfloat16)
    max_tiles = ((P + 127) // 128 + min(E, P)) * (2 * I // 128)
    K_.grouped_gemm(X, d, packed.data_ptr(), P_el * 2, E, 2 * I, offsets=perm["offsets"], active=perm["active"],
                    max_tiles=max_tiles, epi=K_.GG_SWIGLU_BF16, out_bf16=U, ldo=I)
    Y = torch.full((P, d), float("nan"), device=dev)
    max_tiles = ((P + 127) // 128 + min(E, P)) * (d // 128)
    K_.grouped_gemm(U, I, packed.data_ptr() + w13_el * 2, P_el * 2, E, d, offsets=perm["offsets"],
                    active=perm["active"], max_tiles=max_tiles, epi=K_.GG_STORE_F32, out_f32=Y, ldo=d,
                    row_to_pair=perm["sorted_pairs"])
    torch.cuda.synchronize()
    # reference on the same bf16 operands, U rounded to bf16 like the kernel
    xb = h2.bfloat16().float()
    w1, w3, w2 = w_in.bfloat16().float(), w_up.bfloat16().float(), w_out.bfloat16().float()
    idx_c = idx.long()
    for p in range(0, P, max(1, P // 64)):
        t, j = divmod(p, k)
        e = int(idx_c[t, j])
        gte = xb[t] @ w1[e]
        up = xb[t] @ w3[e]
        u = (torch.nn.functional.silu(gte) * up).bfloat16().float()
        want = u @ w2[e]
        assert rel_err(Y[p].cpu().numpy(), want.cpu().numpy()) < 1e-2, p
    assert not torch.isnan(Y).any()
