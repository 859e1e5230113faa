"""Expert-parallel layer on one GPU (world size 1): the single-GPU MoBiLE
layer vs the peer-memory EP layer (ep_p2p.cu exchange kernels around the same
experts) vs the NCCL-path EP layer; CUDA-event time per layer call.
    python scripts/bench_ep.py [preset] [T...]"""
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.ep import ExpertParallelMoE, P2PExpertParallelMoE  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel, MoBiLEMoE  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
Ts = [int(t) for t in sys.argv[2:]] or [1, 8, 64]
spec = replace(PRESETS[name], num_layers=2)
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
E, d, k = spec.num_experts, spec.hidden_dim, spec.k_big
local = MoBiLEMoE(dm.dw.shard_experts(0, E))
out = {}
for T in Ts:
    x = torch.randn(T, d, device="cuda")
    k_tok = torch.full((T,), k, dtype=torch.int32, device="cuda")
    p2p = P2PExpertParallelMoE(dm.moe, local, E, d, cap=T * k)
    nccl = ExpertParallelMoE(dm.moe, local, E)
    fns = {"single_gpu": lambda: dm.moe.forward(x, 0, k_tok, k),
           "ep_p2p_world1": lambda: p2p.forward(x, 0, k_tok, k),
           "ep_nccl_path_world1": lambda: nccl.forward(x, 0, k_tok, k)}
    row = {}
    for kname, fn in fns.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        row[kname] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    p2p.x.close()
    out[f"T{T}"] = row
    print(name, T, row, flush=True)
print(json.dumps({"model": name, "us_per_layer": out,
                  "note": "world size 1: the exchange kernels' own cost (no NVLink traffic); the NCCL-path "
                          "layer at world 1 degenerates to local copies + its host syncs"}))
