"""Repro helper: build a large-batch (GEMM path) StepEngine and replay its passes.
    python scripts/debug_gemm_batch.py PRESET B LAYERS MAX_LEN"""
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name, B, L, ml = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
spec = PRESETS[name] if L <= 0 else replace(PRESETS[name], num_layers=L)
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
if "--garbage" in sys.argv:  # leave stale bytes (NaN floats / -1 ints) in the allocator's cached blocks
    junk = [torch.full((1 << 28,), -1, dtype=torch.int32, device="cuda") for _ in range(40)]
    del junk
eng = StepEngine(dm, B, ml, graphs="--eager" not in sys.argv).build()
torch.cuda.synchronize()
print("built", flush=True)
for kd in ("little", "big", "full"):
    eng.pass_resident(kd)
    torch.cuda.synchronize()
    print(kd, "ok", flush=True)
