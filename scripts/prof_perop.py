"""One graph-free little pass of the per-op engine (batch 1, resident, context
512) for an ncu launch list.  python scripts/prof_perop.py [c3]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

spec = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 560, graphs=False, persistent=False).build()
eng.sess.kc.normal_()
eng.sess.vc.normal_()
eng.pos.fill_(512)
torch.cuda.synchronize()
eng.run_pass("little")
torch.cuda.synchronize()
print("ok")
