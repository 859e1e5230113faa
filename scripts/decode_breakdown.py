"""Where does a decode token's time go?  Qwen shape, batch 1:
resident experts (one graph per pass) vs offloaded experts with a cache that
holds everything (pure per-layer protocol overhead) vs the 477-slot cache."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.offload import OffloadRuntime  # noqa: E402
from paper_2510_12357_b200.presets import QWEN15_MOE  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

dev = torch.device("cuda")
spec = QWEN15_MOE
out = {}
rng = np.random.default_rng(0)
stream_ids = rng.integers(1, spec.vocab_size, size=200).tolist()
prompt = rng.integers(1, spec.vocab_size, size=64).tolist()


XFER = {}


def run(eng, n, full=False, flags=None):
    eng.prefill(prompt)
    for i in range(8):
        eng.step(False, full=full, next_token=stream_ids[i])
    torch.cuda.synchronize()
    x0 = eng.rt.counters()[1] if eng.rt else 0
    t0 = time.perf_counter()
    for i in range(8, 8 + n):
        eng.step(False if flags is None else flags[i], full=full, next_token=stream_ids[i])
    torch.cuda.synchronize()
    XFER["last"] = ((eng.rt.counters()[1] if eng.rt else 0) - x0) / n
    return (time.perf_counter() - t0) / n * 1e3


dw = DeviceWeights.random(spec, dev, seed=0)
dm = DeviceModel(dw)
eng = StepEngine(dm, 1, 256).build()
out["resident_little_ms"] = round(run(eng, 32), 3)
out["resident_full_ms"] = round(run(eng, 32, full=True), 3)
out["resident_mobile_r100_ms"] = round(run(eng, 32, flags=[True] * 64), 3)
# GPU-only time of one pass graph (replayed back to back on the engine stream)
for kd in ("little", "full"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(eng.stream):
        e0.record()
        for _ in range(20):
            eng.graphs[kd].replay()
        e1.record()
    torch.cuda.synchronize()
    out[f"resident_{kd}_graph_gpu_ms"] = round(e0.elapsed_time(e1) / 20, 3)
del eng, dm, dw
torch.cuda.empty_cache()

dw = DeviceWeights.random(spec, dev, seed=0, experts_on_device=False)
dm = DeviceModel(dw)
for slots in (1440, 477):
    rt = OffloadRuntime(dw, slots)
    eng = StepEngine(dm, 1, 256, runtime=rt).build()
    run(eng, 16)  # warm the cache
    out[f"offload{slots}_little_ms"] = round(run(eng, 32), 3)
    out[f"offload{slots}_little_xfer_per_tok"] = round(XFER["last"], 2)
    out[f"offload{slots}_little_pcie_ms_at_55GBs"] = round(XFER["last"] * dw.expert_bytes / 55e9 * 1e3, 3)
    out[f"offload{slots}_full_ms"] = round(run(eng, 32, full=True), 3)
    out[f"offload{slots}_full_xfer_per_tok"] = round(XFER["last"], 2)
    out[f"offload{slots}_full_pcie_ms_at_55GBs"] = round(XFER["last"] * dw.expert_bytes / 55e9 * 1e3, 3)
    del eng, rt
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
