"""One prefill (per-op engine) for an ncu launch list (the second prefill,
between cudaProfilerStart/Stop):
    ncu --profile-from-start off --metrics gpu__time_duration.sum ... python scripts/prof_prefill.py c5 2048"""
import sys
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
prompt = np.random.default_rng(0).integers(1, spec.vocab_size, size=n + 1).tolist()
eng.prefill(prompt)  # warm-up
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only the second prefill
eng.prefill(prompt)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
