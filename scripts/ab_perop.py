"""A/B of the per-op (resident, batch-1) engine: graph-replayed pass times.
    python scripts/ab_perop.py c3 [tag]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
tag = sys.argv[2] if len(sys.argv) > 2 else "default"
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 600, persistent=False).build()
eng.sess.kc.normal_()
eng.sess.vc.normal_()
eng.pos.fill_(512)
torch.cuda.synchronize()
out = {"tag": tag, "model": name}
for kd in ("little", "full"):
    best = 1e9
    for rep in range(3):
        eng.graphs[kd].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            e0.record()
            for _ in range(20):
                eng.graphs[kd].replay()
            e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
    out[kd] = round(best, 1)
    out[kd + "_states_sum"] = float(eng.states[kd].double().abs().sum())
print(json.dumps(out), flush=True)
