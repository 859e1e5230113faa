"""Per-phase timeline of one persistent decode pass (globaltimer trace):
barrier latency, input-build time and work time per phase kind."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200 import _native as N  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
kind = sys.argv[2] if len(sys.argv) > 2 else "little"
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 600, graphs=False, persistent=True).build()
info = eng.dp_info(kind)
G, nph = info["grid"], info["phases"]
trace = torch.zeros(nph * G * 6, dtype=torch.int64, device="cuda")
prompt = np.random.default_rng(0).integers(1, spec.vocab_size, size=512).tolist()
eng.prefill(prompt)
for i in range(3):
    eng.step(False, next_token=i + 5)
N.lib.mobile_dp_set_trace(eng.dp[kind], trace.data_ptr())
torch.cuda.synchronize()
with torch.cuda.stream(eng.stream):
    eng.run_pass(kind)
torch.cuda.synchronize()
t = trace.view(nph, G, 6).cpu().numpy().astype(np.float64)
t0 = t[0, :, 0].min()
t = (t - t0) / 1e3  # us
names = ["qkv", "attn", "o", "router+sgu", "gu+sd", "down"]
per = {}
prev_done = 0.0
rows = []
for p in range(nph):
    kindname = "head" if p == nph - 1 else names[p % 6]
    start_max = t[p, :, 0].max()
    ready_max = t[p, :, 1].max()
    done = t[p, :, 2]
    done_max = done.max() if p < nph - 1 else float("nan")
    rows.append((p, kindname, round(start_max, 2), round(ready_max, 2), round(done_max, 2)))
    d = per.setdefault(kindname, dict(n=0, bar=0.0, ready=0.0, work=0.0, release=0.0, observe=0.0, acquire=0.0))
    d["n"] += 1
    d["bar"] += start_max - prev_done
    if p > 0:  # the barrier this phase waited on: previous phase's arrivals
        q = p - 1
        d["release"] += float(np.max(t[q, :, 3] - t[q, :, 2]))          # slowest red.release issue
        d["observe"] += float(np.median(t[p, :, 4]) - t[q, :, 3].max())  # last arrival -> median observer
        d["acquire"] += float(np.max(t[p, :, 5] - t[p, :, 4]))         # slowest acquire fence
    d["ready"] += ready_max - start_max
    if p < nph - 1:
        d["work"] += done_max - ready_max
        prev_done = done_max
out = {k: {kk: round(vv, 1) if isinstance(vv, float) else vv for kk, vv in v.items()} for k, v in per.items()}
print(json.dumps(dict(model=name, kind=kind, info=info, per_kind=out, first_phases=rows[:14], last=rows[-3:]), indent=1))
