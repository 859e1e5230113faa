"""Debug: max / total time of the early-route computation (build with -DMOBILE_DP_TIME_ROUTE)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200 import _native as N  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

spec = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
eng = StepEngine(dm, 1, 600, persistent=True).build()
eng.pos.fill_(512)
for _ in range(3):
    eng.run_pass("little")
torch.cuda.synchronize()
d = (C.c_int * 16)()
N.lib.mobile_dp_diag(eng.dp["little"], d)
print("route ns max", d[14], "sum", d[15], "second call: max", d[12], "sum", d[13], "calls", spec.num_layers * (3 + 1), "sections load/rank/topk+softmax/permute/tail", list(d)[4:9])
