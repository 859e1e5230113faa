"""Isolated timing of the bulk-copy streaming GEMV (dense STORE groups and the
head) at decode sizes, L2-cold (rotating through matrices > L2)."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
res = {}
for rows, Kd in ((2048, 2048), (6144, 2048), (16896, 2048), (151936, 2048), (524288, 2048), (2048, 5632)):
    nbytes = rows * Kd * 2
    nmat = max(2, int(2.0e9 // nbytes))  # rotate through >= 2 GB of weights
    mats = [torch.randn(rows, Kd, device=dev).to(torch.bfloat16) for _ in range(min(nmat, 64))]
    x = torch.randn(1, Kd, device=dev)
    out = torch.empty(1, rows, device=dev)
    def run(i):
        w = mats[i % len(mats)]
        K.stream_gemv([K.sg_group(w_base=w.data_ptr(), K=Kd, rows=rows, x=x, dense_T=1, out=out)], 1, 1)
    for i in range(3):
        run(i)
    torch.cuda.synchronize()
    reps = 2 * len(mats)
    # capture the launches in a CUDA graph so host launch overhead is excluded
    s_ = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s_):
        run(0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s_):
        for i in range(reps):
            run(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    res[f"store_{rows}x{Kd}"] = dict(MB=round(nbytes / 1e6, 1), us=round(us, 2), GBs=round(nbytes / us / 1e3, 1),
                                     frac=round(nbytes / us / 1e3 / peak, 3))
    del mats
    torch.cuda.empty_cache()
# head mode at the Qwen vocabulary
V, d = 151936, 2048
mats = [torch.randn(V, d, device=dev).to(torch.bfloat16) for _ in range(4)]
ws = K.StreamHeadWorkspace(dev)
x = torch.randn(1, d, device=dev)
for i in range(3):
    K.stream_head(x, mats[i % 4], 0.5, 24.0, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(8):
    K.stream_head(x, mats[i % 4], 0.5, 24.0, ws=ws)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 8 * 1e3
res["head_151936x2048"] = dict(us=round(us, 2), GBs=round(V * d * 2 / us / 1e3, 1), frac=round(V * d * 2 / us / 1e3 / peak, 3))
print(json.dumps(res, indent=1))
