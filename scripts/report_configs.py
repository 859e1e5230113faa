"""Per-config report (BASELINE.json configs C2-C5, 1 GPU, experts HBM-resident):
decode pass times of the persistent kernel for the little / replayed big /
full-top-k passes, MoBiLE tokens/s at the paper's fallback ratio vs the
full-top-k baseline, each pass's HBM roofline fraction; prefill tokens/s
(per-op engine: tcgen05 grouped GEMM experts) with the expert GEMMs' tensor
roofline fraction.  Writes JSON to stdout (profiles/r1_configs.json).

    python scripts/report_configs.py [c2 c3 c4 c5]
"""
import json
import math
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402
from paper_2510_12357_b200.presets import NAMES, PRESETS  # noqa: E402
from paper_2510_12357_b200.runtime import StepEngine  # noqa: E402
from paper_2510_12357_b200.weights import DeviceWeights  # noqa: E402

PK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
R_PAPER = {"c2": 0.21, "c3": 0.11, "c4": 0.11, "c5": 0.11}  # PAPER.md fallback ratios (OLMoE 0.21, Qwen 0.11)
PROMPT = {"c2": 512, "c3": 512, "c4": 512, "c5": 2048}
BATCHES = {"c4": (1, 2, 4, 8, 64, 256)}


def pass_bytes(spec, dw, kind_k, ctx, B):
    eb, d, L = dw.elem_bytes, spec.hidden_dim, spec.num_layers
    experts = min(spec.num_experts, B * kind_k) * dw.expert_bytes
    per_layer = (2 * d * d + 2 * d * spec.kv_dim + (spec.num_experts + dw.n_gate_rows) * d) * eb + experts + spec.n_shared * dw.shared_bytes \
        + B * 2 * ctx * spec.kv_dim * 4
    return L * per_layer + spec.vocab_size * d * eb


def time_graph(eng, kind, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(eng.stream):
        e0.record()
        for _ in range(reps):
            eng.graphs[kind].replay()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


out = {"peaks": {"hbm_gbs": PK["hbm_gbs"], "bf16_tflops": PK["bf16_tflops"]}}
for name in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
    spec = PRESETS[name]
    if os.environ.get("REPORT_LAYERS"):  # debugging: fewer layers
        spec = replace(spec, num_layers=int(os.environ["REPORT_LAYERS"]))
    t0 = time.time()
    dw = DeviceWeights.random(spec, torch.device("cuda"), seed=0)
    dm = DeviceModel(dw)
    res = {"model": NAMES[name], "init_s": round(time.time() - t0, 1), "decode": {}}
    ctx = PROMPT[name]

    def engine(B, gemm=None):
        e = StepEngine(dm, B, ctx + 48, gemm=gemm).build()
        # B sequences at a common position: fill the caches with random K/V rows
        e.sess.kc.normal_()
        e.sess.vc.normal_()
        e.pos.fill_(ctx)
        e.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32))
        for kd in ("little", "big", "full"):
            e.graphs[kd].replay()
        torch.cuda.synchronize()
        return e

    r = R_PAPER[name]
    batches = BATCHES.get(name, (1,))
    if os.environ.get("REPORT_BATCHES"):
        batches = tuple(int(b) for b in os.environ["REPORT_BATCHES"].split(","))
    for B in batches:
        print(f"[{name}] B={B}", file=sys.stderr, flush=True)
        eng = engine(B)
        row = {"path": "gemm" if eng.gemm_path else ("persistent" if eng.dp else "per-op")}
        if eng.dp:
            row["dp_info"] = eng.dp_info()
        for kd in ("little", "big", "full"):
            t = time_graph(eng, kd)
            nb = pass_bytes(spec, dw, eng.k[kd], ctx, B)
            row[kd] = {"ms": round(t * 1e3, 3), "bytes": nb, "gbs": round(nb / t / 1e9, 1),
                       "hbm_frac": round(nb / t / 1e9 / PK["hbm_gbs"], 3)}
        del eng
        torch.cuda.empty_cache()
        # batched MoBiLE: the big pass replays only the rows that fell back.
        # P(any row falls back) = 1 - (1 - r)^B; given that, E[rows] = rB / P.
        p_any = 1.0 - (1.0 - r) ** B
        b_fb = max(1, math.ceil(r * B / p_any - 1e-9))
        if b_fb == B:
            t_big = row["big"]["ms"]
        else:
            e2 = engine(b_fb)
            t_big = round(time_graph(e2, "big") * 1e3, 3)
            del e2
            torch.cuda.empty_cache()
        row["big_rows"] = {"rows": b_fb, "ms": t_big, "p_any_fallback": round(p_any, 4)}
        t_mob = row["little"]["ms"] + p_any * t_big
        row["mobile_tokens_s"] = round(B * 1e3 / t_mob, 2)
        row["full_topk_tokens_s"] = round(B * 1e3 / row["full"]["ms"], 2)
        row["speedup_vs_full_topk"] = round(row["full"]["ms"] / t_mob, 4)
        row["r"] = r
        row["note"] = ("tokens/s = B / (T_l(B) + P_any T_b(rows)), T from graph-replayed passes, ctx %d; the big "
                       "pass replays the fallback rows only (batch of E[rows | any])" % ctx)
        res["decode"][f"B{B}"] = row
    # prefill: the per-op engine (attention + tcgen05 grouped-GEMM experts) over the prompt
    sess_eng = StepEngine(dm, 1, ctx + 8, persistent=False)
    prompt = np.random.default_rng(0).integers(1, spec.vocab_size, size=ctx + 1).tolist()
    sess_eng.prefill(prompt)  # warm-up (TMA maps, scratch)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sess_eng.prefill(prompt)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t1
    I, Is, d = spec.ffn, spec.shared_ffn, spec.hidden_dim
    moe_flops = 2.0 * ctx * spec.num_layers * (spec.k_big * 3 * d * I + spec.n_shared * 3 * d * Is)
    res["prefill"] = {"tokens": ctx, "ms": round(tp * 1e3, 2), "tokens_s": round(ctx / tp, 1),
                      "expert_gemm_tflop": round(moe_flops / 1e12, 3),
                      "expert_tflops_whole_prefill": round(moe_flops / tp / 1e12, 1),
                      "note": "wall clock of the full prefill (attention in torch, experts on the tcgen05 grouped "
                              "GEMM); the GEMM kernel alone: scripts/bench_gemm.py"}
    out[name] = res
    print(json.dumps({name: res}), flush=True)
    del sess_eng, dm, dw
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
