"""A/B of decode-pass builds: GPU time of one resident little / full pass
(graph replay, 20 reps) on a preset, for the library named by MOBILE_LIB.
    MOBILE_LIB=... python scripts/ab_dp.py c3 [tag]"""
import json
import os
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

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
tag = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("MOBILE_LIB", "default")
spec = PRESETS[name]
dw = DeviceWeights.random(spec, torch.device("cuda"), seed=0)
dm = DeviceModel(dw)
eng = StepEngine(dm, 1, 600, persistent=True).build()
eng.prefill(np.random.default_rng(0).integers(1, spec.vocab_size, size=512).tolist())
for i in range(3):
    eng.step(False, next_token=i + 5)
out = {"tag": tag, "model": name}
for kd in ("little", "full"):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            e0.record()
            for _ in range(20):
                eng.graphs[kd].replay()
            e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 20 * 1e3)
    out[kd] = round(min(ts), 1)
out["flags"] = int(eng.dp_flags.item())
print(json.dumps(out), flush=True)
