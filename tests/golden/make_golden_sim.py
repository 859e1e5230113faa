"""Golden vectors for the timing model, metrics and traces,
from the UNMODIFIED reference package (`moesim`), imported read-only from
/root/reference/pkg/src in the build container:

    python tests/golden/make_golden_sim.py

Writes tests/golden/sim_golden.json and tests/golden/trace_small.jsonl
(committed; nothing on the GPU box reads /root/reference)."""

from __future__ import annotations

import io
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
from moesim import config as C  # noqa: E402
from moesim import engine as E  # noqa: E402
from moesim import metrics as M  # noqa: E402
from moesim import trace as T  # noqa: E402

out: dict = {}
# a small synthetic workload with tight HBM so the cache evicts and defers
cfg = T.SyntheticTraceConfig(seed=3, num_layers=4, num_experts=16, k_big=4, popularity_skew=0.8, reuse_prob=0.3)
recs = T.gen_synthetic(cfg, 40)
T.save_trace(OUT / "trace_small.jsonl", recs)
model = C.ModelSpec(num_layers=4, num_experts=16, k_big=4, k_little=2, expert_bytes=10 * 1024**2,
                    dense_bytes_per_layer=1024**2)
hw = C.HardwareSpec(hbm_capacity=12 * 10 * 1024**2 + 4 * 1024**2 + 1024**2, reserved=1024**2,
                    pcie_bandwidth=16 * 1024**3, pcie_fixed_latency=1e-4, gpu_expert_compute=3e-4,
                    gpu_attn_compute=2.7e-3, lookahead_depth=2)
out["slots"] = C.hbm_expert_slots(model, hw)
costs = C.derive_costs(model, hw)
out["costs"] = [costs.t_xfer, costs.t_exp, costs.t_attn]
pol = C.PolicySpec(gamma=0.7)
for name, flags in (("conf", None), ("inject", E.injected_fallback_flags(len(recs), 0.3))):
    base, prim, row = M.run_pair(recs, model, hw, pol, fallback_flags=flags)
    out[f"pair_{name}"] = {
        "row": [float(v) for v in row.row()],
        "base_totals": [t.total for t in base],
        "prim": [[[p.label, p.total, p.compute, p.transfer_stall, p.overlapped_transfer, p.fresh_transfers,
                   p.hits, p.misses] for p in t.passes] for t in prim],
        "prim_fallback": [t.fallback for t in prim],
    }
full_mobile, _ = E.simulate_full_stream(recs, costs, out["slots"], 4, plan_mode=E.PLAN_MOBILE, lookahead=2)
out["full_mobile_totals"] = [t.total for t in full_mobile]
out["gamma_sweep"] = [[float(v) for v in r.row()] for r in M.gamma_sweep(recs, model, hw, pol, [0.0, 0.5, 0.7, 1.0])]
out["little_sweep"] = [[float(v) for v in r.row()] for r in M.little_size_sweep(recs, model, hw, pol, [1, 2, 3, 4])]
with tempfile.TemporaryDirectory() as d:
    M.write_metrics_csv(Path(d) / "m.csv", M.gamma_sweep(recs, model, hw, pol, [0.5, 0.9]))
    out["csv"] = (Path(d) / "m.csv").read_text()
out["analytic"] = [M.analytic_speedup(2.0, 1.0, 2.5, 0.2), M.analytic_speedup(3.0, 1.5, 0.0, 0.0)]
cal = T.calibration_trace()
out["calibration"] = {"n": len(cal), "first": cal[0].layers[0, :8].tolist(), "conf0": cal[0].confidence,
                      "sum": float(sum(r.layers.sum() for r in cal)), "conf_sum": float(sum(r.confidence for r in cal))}
events: list = []
M.run_pair(recs[:3], model, hw, pol, event_log=events)
out["events"] = [[t, k, e, l] for t, k, e, l in events]
(OUT / "sim_golden.json").write_text(json.dumps(out))
print("wrote", OUT / "sim_golden.json", len(json.dumps(out)), "bytes")
