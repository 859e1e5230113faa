"""GPU time of one decode pass (graph replay), persistent kernel vs per-op
kernels, resident experts, batch 1; algorithmic bytes per pass and HBM frac."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
res = {}
for name in sys.argv[1:] or ["c3", "c2"]:
    spec = PRESETS[name]
    dw = DeviceWeights.random(spec, torch.device("cuda"), seed=0)
    dm = DeviceModel(dw)
    eb = dw.elem_bytes
    d, L = spec.hidden_dim, spec.num_layers
    ctx = 512
    for persistent in (True, False):
        eng = StepEngine(dm, 1, ctx + 64, persistent=persistent).build()
        prompt = np.random.default_rng(0).integers(1, spec.vocab_size, size=ctx).tolist()
        eng.prefill(prompt)
        for i in range(3):
            eng.step(False, next_token=i + 5)
        for kd in ("little", "big", "full"):
            k = eng.k[kd]
            per_layer = (2 * d * d + 2 * d * spec.kv_dim + (spec.num_experts + dw.n_gate_rows) * d) * eb + k * dw.expert_bytes \
                + spec.n_shared * dw.shared_bytes + 2 * ctx * spec.kv_dim * 4
            tot = L * per_layer + spec.vocab_size * d * eb
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(eng.stream):
                e0.record()
                for _ in range(20):
                    eng.graphs[kd].replay()
                e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            res[f"{name}_{'dp' if persistent else 'perop'}_{kd}"] = dict(
                us=round(us, 1), MB=round(tot / 1e6, 1), GBs=round(tot / us / 1e3, 1),
                frac=round(tot / us / 1e3 / peak, 3))
        if persistent:
            res[f"{name}_dp_info"] = eng.dp_info()
            res[f"{name}_dp_flags"] = int(eng.dp_flags.item())
        del eng
        torch.cuda.empty_cache()
    del dm, dw
    torch.cuda.empty_cache()
    print(json.dumps(res, indent=1), flush=True)
