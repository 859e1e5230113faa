"""Wall time of one prefill of n tokens (second call; per-op engine).
    python scripts/time_prefill.py c5 2048"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, n + 8, persistent=False)
prompt = np.random.default_rng(1).integers(1, spec.vocab_size, size=n).tolist()
ts = []
for _ in range(4):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    eng.prefill(prompt)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - w0)
print(name, n, "prefill ms", [round(t * 1e3, 2) for t in ts], flush=True)
