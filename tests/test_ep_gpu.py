"""Expert-parallel layer on the device (world size 1 here: one GPU per gpurun);
the multi-rank exchange is covered by tests/test_ep_cpu.py over gloo."""
import numpy as np
import pytest
import torch

from tests.helpers import QWEN_MINI, matched

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T", [1, 3, 40])
def test_ep_layer_equals_single_gpu_layer(cuda_ok, T):
    from paper_2510_12357_b200.ep import ExpertParallelMoE
    from paper_2510_12357_b200.model import MoBiLEMoE
    o, ms, dm = matched(QWEN_MINI, "bfloat16")
    dw = dm.dw
    local = MoBiLEMoE(dw.shard_experts(0, ms.num_experts))
    ep = ExpertParallelMoE(dm.moe, local, ms.num_experts)
    rng = np.random.default_rng(T)
    x = torch.tensor(rng.normal(size=(T, ms.hidden_dim)), dtype=torch.float32, device="cuda")
    k_tok = torch.tensor(rng.choice([ms.k_little, ms.k_big], size=T), dtype=torch.int32, device="cuda")
    want, _ = dm.moe.forward(x, 0, k_tok, ms.k_big)
    want = want.clone()
    got = ep.forward(x, 0, k_tok, ms.k_big)
    # identical kernels when both sides stream (fp32 activations); once either side has >= 5
    # rows it runs the tcgen05 GEMM on bf16 activations -> the bf16 bar
    bf16_path = T >= 5 or int(k_tok.sum()) >= 5
    err = (got - want).abs().max().item() / want.abs().max().item()
    assert err < (2e-2 if bf16_path else 1e-5), err
