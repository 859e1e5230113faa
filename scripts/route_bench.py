"""Debug: cycles of compute_route alone (variant lib built with -DMOBILE_DP_ROUTE_BENCH)."""
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

for name in sys.argv[1:] or ["c3"]:
    spec = PRESETS[name]
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
    eng = StepEngine(dm, 1, 600, persistent=True).build()
    eng.pos.fill_(512)
    eng.run_pass("little")
    torch.cuda.synchronize()
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for kd in ("little", "full"):
        N.lib.mobile_dp_route_bench(eng.dp[kd], 200, C.c_void_p(out.data_ptr()))
        print(name, kd, "cycles per compute_route", int(out.item()))
