"""Per-step error anatomy of the full-width parity case (debug)."""
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import moe_ref as R  # noqa: E402
from tests.fullshape import device_oracle  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

preset, layers, persistent = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
spec = replace(PRESETS[preset], num_layers=layers)
dw = DeviceWeights.random(spec, torch.device("cuda"), seed=21)
eng = StepEngine(DeviceModel(dw), 1, 64, persistent=persistent).build(gamma=0.7)
W = device_oracle(dw)
rng = np.random.default_rng(5)
prompt = rng.integers(1, spec.vocab_size, size=int(sys.argv[4]) if len(sys.argv) > 4 else 4).tolist()
dec = R.KVDecoder(W)
dec.prefill(prompt[:-1])
eng.prefill(prompt)
for i in range(3):
    eng.step(forced_fallback=False, next_token=prompt[-1])
    probs, states, sel, kv = dec.run([prompt[-1] if i == 0 else prompt[-1]], spec.k_little)
    dec.commit(kv)
    g = eng.states["little"][:, 0].cpu().numpy()
    per_layer = np.abs(g - states).max(axis=1) / np.abs(states).max(axis=1)
    conf = eng.head["little"]["conf"].item()
    print(i, "state err per layer", per_layer, "conf", conf, probs.max(), "argmax", eng.head["little"]["argmax"].item(), probs.argmax())
