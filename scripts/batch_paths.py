"""Decode pass time per batch: persistent pass vs GEMM path vs per-op GEMV
engine (the measurements behind StepEngine's defaults).
    python scripts/batch_paths.py [preset] [B...]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
batches = [int(b) for b in sys.argv[2:]] or [1, 2, 3, 4]
spec = PRESETS[name]
dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=0))
out = {}
for B in batches:
    modes = ([(False, True)] if B <= 4 else []) + [(True, None)] + ([(False, False)] if B <= 4 else [])
    for gemm, persistent in modes:
        eng = StepEngine(dm, B, 560, gemm=gemm, persistent=persistent).build()
        eng.sess.kc.normal_()
        eng.sess.vc.normal_()
        eng.pos.fill_(512)
        # random token ids (as bench.py): distinct rows route to distinct experts
        eng.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32,
                                    generator=torch.Generator("cuda").manual_seed(B)))
        torch.cuda.synchronize()
        res = {}
        for kd in ("little", "full"):
            eng.graphs[kd].replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(eng.stream):
                e0.record()
                for _ in range(10):
                    eng.graphs[kd].replay()
                e1.record()
            torch.cuda.synchronize()
            res[kd] = round(e0.elapsed_time(e1) / 10, 3)
        name_ = "gemm" if gemm else ("persistent" if persistent else "perop_gemv")
        out[f"B{B}_{name_}"] = res
        print(B, name_, res, flush=True)
        del eng
        torch.cuda.empty_cache()
print(json.dumps(out))
