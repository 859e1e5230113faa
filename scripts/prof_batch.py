"""One eager large-batch decode pass (GEMM path) for an ncu launch list.
    ncu --metrics gpu__time_duration.sum --csv python scripts/prof_batch.py c4 64 little"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name, B, kind = sys.argv[1], int(sys.argv[2]), sys.argv[3]
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, B, 560, graphs=False).build()
eng.sess.kc.normal_()
eng.sess.vc.normal_()
eng.pos.fill_(512)
eng.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32))
torch.cuda.synchronize()
eng.run_pass(kind)
torch.cuda.synchronize()
print("ok")
