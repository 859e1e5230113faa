"""Kernel microbenchmark at the Qwen1.5-MoE decode shapes (batch 1).

Times, with CUDA events over many launches whose weights span > L2 (all 24
layers distinct), the expert gate-up and down launches of one MoE layer
(routed little k=2 + the 5632-wide shared expert), for the bulk-copy streaming
kernel and the warp-streaming kernel, and the head GEMV.  Prints GB/s and the
fraction of MEASURED_PEAKS hbm_gbs.
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2510_12357_b200 import kernels as K  # noqa: E402
from paper_2510_12357_b200 import model as M  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import QWEN15_MOE, OLMOE  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
dev = torch.device("cuda")
out = {}
for name, spec in (("qwen", QWEN15_MOE), ("olmoe", OLMOE)):
    dw = DeviceWeights.random(spec, dev, seed=0)
    dm = DeviceModel(dw)
    moe = dm.moe
    L, d = spec.num_layers, spec.hidden_dim
    x = torch.randn(1, d, device=dev)
    for kname, k in (("little", spec.k_little), ("big", spec.k_big)):
        k_tok = torch.full((1,), k, dtype=torch.int32, device=dev)
        scs = [moe.route(x, l, k_tok, k) for l in range(L)]
        scs = [dict(sc) for sc in scs]  # route() returns views of shared scratch: rebuild per layer
        for impl in ("stream",):
            M.FFN_IMPL = impl
            try:
                sc0 = moe.route(x, 0, k_tok, k)
                moe.experts(x, 0, sc0, k_tok, k)
            except Exception as exc:  # warp kernels need row-major (untiled) K
                out[f"{name}_{kname}_{impl}"] = f"n/a: {exc}"
                continue
            for it in range(3):
                for l in range(L):
                    sc = moe.route(x, l, k_tok, k)
                    moe.experts(x, l, sc, k_tok, k)
            torch.cuda.synchronize()
            # time the whole expert block (gate-up + down + combine) per layer
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n_rep = 5
            sc_l = [moe.route(x, l, k_tok, k) for l in range(1)]
            e0.record()
            for rep in range(n_rep):
                for l in range(L):
                    sc = moe.route(x, l, k_tok, k)
                    moe.experts(x, l, sc, k_tok, k)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / (n_rep * L)
            nbytes = k * dw.expert_bytes + spec.n_shared * dw.shared_bytes + (E := spec.num_experts) * d * 2
            out[f"{name}_{kname}_{impl}_layer_us"] = round(ms * 1e3, 2)
            out[f"{name}_{kname}_{impl}_GBs"] = round(nbytes / (ms / 1e3) / 1e9, 1)
            out[f"{name}_{kname}_{impl}_frac"] = round(nbytes / (ms / 1e3) / 1e9 / peak, 3)
    del dw, dm, moe
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "bench_kernels.json").write_text(json.dumps(out, indent=1))
