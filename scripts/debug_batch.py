"""B=2 decode pass vs two B=1 passes, persistent and per-op engines."""
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

spec = replace(PRESETS[sys.argv[1] if len(sys.argv) > 1 else "c4"], num_layers=2)
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=4))
B, ctx = 2, 37
g = torch.Generator(device="cuda").manual_seed(0)
e2 = StepEngine(dm, B, 64, persistent=True).build()
kc = torch.randn(e2.sess.kc.shape, device="cuda", generator=g)
vc = torch.randn(e2.sess.vc.shape, device="cuda", generator=g)
tok = torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32, generator=g)
for persistent in (True, False):
    eb = StepEngine(dm, B, 64, persistent=persistent).build()
    e1 = StepEngine(dm, 1, 64, persistent=persistent).build()
    eb.sess.kc.copy_(kc); eb.sess.vc.copy_(vc); eb.pos.fill_(ctx); eb.tok.copy_(tok)
    eb.run_pass("little")
    torch.cuda.synchronize()
    for s in range(B):
        e1.sess.kc.copy_(kc[:, s:s + 1]); e1.sess.vc.copy_(vc[:, s:s + 1]); e1.pos.fill_(ctx); e1.tok.copy_(tok[s:s + 1])
        e1.run_pass("little")
        torch.cuda.synchronize()
        for l in range(spec.num_layers):
            a = eb.states["little"][l, s].cpu().numpy()
            b = e1.states["little"][l, 0].cpu().numpy()
            print("persistent" if persistent else "per-op", "seq", s, "layer", l, "max|d|", float(np.abs(a - b).max()),
                  "idx", eb.idx["little"][l, s].tolist(), e1.idx["little"][l, 0].tolist())
        print("   conf", float(eb.head["little"]["conf"][s]), float(e1.head["little"]["conf"][0]),
              "argmax", int(eb.head["little"]["argmax"][s]), int(e1.head["little"]["argmax"][0]))
    del eb, e1
