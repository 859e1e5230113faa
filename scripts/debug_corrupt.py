"""Repro helper: do persistent-pass engines (B = 1, 2, 4) leave the shared
weights untouched?  python scripts/debug_corrupt.py PRESET LAYERS MAX_LEN B..."""
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name, L, ml = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = PRESETS[name] if L <= 0 else replace(PRESETS[name], num_layers=L)
dw = DeviceWeights.random(spec, torch.device("cuda"), seed=0)
dm = DeviceModel(dw)
names = ("embed", "qkv", "o", "router", "experts", "shared", "head")


def sums():
    return {n: float(getattr(dw, n).double().sum()) for n in names if getattr(dw, n) is not None}


ref = sums()
for B in map(int, sys.argv[4:]):
    eng = StepEngine(dm, B, ml, persistent=B <= 4).build()
    eng.sess.kc.normal_()
    eng.sess.vc.normal_()
    eng.pos.fill_(ml - 48)
    eng.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32))
    for kd in ("little", "big", "full"):
        for _ in range(3):
            eng.graphs[kd].replay()
    torch.cuda.synchronize()
    now = sums()
    bad = [n for n in ref if now[n] != ref[n]]
    print("B", B, "flags", int(eng.dp_flags.item()) if eng.dp else None, "changed:", bad,
          "conf", eng.head["little"]["conf"].tolist()[:4], flush=True)
    del eng
    torch.cuda.empty_cache()
