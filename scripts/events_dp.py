"""Per-CTA event timeline of one persistent decode pass (producer issues,
consumer stage waits, phase barriers) for one layer of CTA `cta`."""
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

spec = PRESETS["c3"]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 600, graphs=False, persistent=True).build()
G = eng.dp_info()["grid"]
ev = torch.zeros(G * 2 * 1024 * 2, dtype=torch.int64, device="cuda")
eng.prefill(np.random.default_rng(0).integers(1, spec.vocab_size, size=512).tolist())
for i in range(3):
    eng.step(False, next_token=i + 5)
N.lib.mobile_dp_set_events(eng.dp["little"], ev.data_ptr())
torch.cuda.synchronize()
with torch.cuda.stream(eng.stream):
    eng.run_pass("little")
torch.cuda.synchronize()
e = ev.view(G, 2, 1024, 2).cpu().numpy()
t0 = e[:, :, 0, 0][e[:, :, 0, 0] > 0].min()
names = {1: "W", 2: "X", 3: "FULL", 4: "UNIT", 5: "ARRIVE", 6: "PASS", 7: "READY", 8: "ROUTE", 9: "WAIT", 10: "RED"}
ppl = 6
for cta in [int(a) for a in (sys.argv[1:] or ["0", "77"])]:
    rows = []
    for role in (0, 1):
        for t, c in e[cta, role]:
            if t == 0:
                continue
            code, ph, item = int(c) >> 56, (int(c) >> 32) & 0xffff, int(c) & 0xffffffff
            rows.append(((t - t0) / 1e3, ("P" if role == 0 else "C"), names.get(code, code), ph, item))
    rows.sort()
    print(f"---- CTA {cta}: layer 1 (phases {ppl}..{2 * ppl})")
    for r in rows:
        if ppl <= r[3] <= 2 * ppl or r[2] == "X":
            if 80 < r[0] < 200:
                print("%8.2f %s %-6s ph=%3d item=%d" % r)
