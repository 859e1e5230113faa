"""Short run for ncu: resident Qwen1.5-MoE shape, persistent decode pass,
prefill 512 then a few little-pass steps (graph replays)."""
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
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 600, persistent=True).build()
eng.prefill(np.random.default_rng(0).integers(1, spec.vocab_size, size=512).tolist())
for i in range(n):
    eng.step(False, next_token=i + 5)
torch.cuda.synchronize()
print("done", eng.dp_info())
