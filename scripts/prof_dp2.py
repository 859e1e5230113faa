"""Short run for ncu DRAM accounting: resident preset, persistent decode pass,
synthetic context of `ctx` positions, `n` graph-replayed passes of `kind`.
    python scripts/prof_dp2.py c3 little 512 3"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name, kind = sys.argv[1], sys.argv[2]
ctx, n = int(sys.argv[3]), int(sys.argv[4])
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, ctx + 64, persistent=True).build()
eng.sess.kc.normal_()
eng.sess.vc.normal_()
eng.pos.fill_(ctx)
torch.cuda.synchronize()
for i in range(n):
    eng.graphs[kind].replay()
torch.cuda.synchronize()
print("done", kind, ctx)
