"""Short resident-expert decode of a real shape, for ncu launch lists / captures.

    python scripts/prof_decode.py [qwen|olmoe] [steps] [graphs 0|1]
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import OLMOE, QWEN15_MOE  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
graphs = bool(int(sys.argv[3])) if len(sys.argv) > 3 else False
spec = {"qwen": QWEN15_MOE, "olmoe": OLMOE}[name]
dev = torch.device("cuda")
dm = DeviceModel(DeviceWeights.random(spec, dev, seed=0))
eng = StepEngine(dm, 1, 256, graphs=graphs).build()
eng.prefill([5, 6, 7, 8])
torch.cuda.synchronize()
for i in range(steps):
    eng.step(forced_fallback=(i % 2 == 1), next_token=100 + i)
torch.cuda.synchronize()
print("done")
