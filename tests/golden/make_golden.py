"""Generate golden vectors from the UNMODIFIED reference package (`moesim`).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `moesim` from /root/reference/pkg/src read-only and writes
`tests/golden/golden.json` + `tests/golden/golden.npz`.  Those fixtures are
committed; nothing at test/bench time on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(REF))
from moesim import config as mconfig  # noqa: E402
from moesim import engine as mengine  # noqa: E402
from moesim import memory as mmemory  # noqa: E402
from moesim import policy as mpolicy  # noqa: E402
from moesim import toymoe as mtoy  # noqa: E402

SPECS = {
    # test_toymoe.py:20-23
    "small": dict(num_layers=3, num_experts=8, k_big=4, k_little=2, hidden_dim=16, vocab_size=32, seed=7),
    # SPEC.md tiny config, BASELINE configs[0] (C1)
    "c1": dict(num_layers=2, num_experts=16, k_big=4, k_little=2, hidden_dim=256, vocab_size=256, seed=0),
    # test_acceptance.py:190-191 (k_little == k_big)
    "a7": dict(num_layers=3, num_experts=8, k_big=4, k_little=4, hidden_dim=16, vocab_size=32, seed=11),
}

arrays: dict[str, np.ndarray] = {}
meta: dict = {"generator": "tests/golden/make_golden.py", "reference": "moesim (pkg/src) @ /root/reference"}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- top_k
rng = np.random.default_rng(3)
topk_cases = []
for i in range(200):  # test_toymoe.py:43-50 tie-forced random cases
    e = int(rng.integers(2, 24))
    k = int(rng.integers(1, e + 1))
    logits = np.round(rng.normal(size=e) * 2) / 2
    topk_cases.append({"logits": logits.tolist(), "k": k, "want": mtoy.top_k(logits, k)})
special = [
    ([0.5, 2.0, 1.0, 3.0], 2), ([1.0, 1.0, 0.0], 1), ([5.0, 5.0, 5.0], 2), ([0.1, -2.0, 3.0, 0.1], 4),
    ([0.0, -0.0, 0.0, -0.0], 4), ([-0.0, 0.0, -1.0], 2), ([0.0, 1e-310, -1e-310, 0.0], 4),
    ([-1e-310, -0.0, 1e-310], 3), ([float(x) for x in range(64)][::-1], 8), ([1.0] * 64, 8),
]
for logits, k in special:
    topk_cases.append({"logits": logits, "k": k, "want": mtoy.top_k(np.array(logits), k)})
# larger rows at the real-shape expert counts, tie-forced
for E in (8, 16, 60, 64, 128, 256):
    for _ in range(20):
        k = int(rng.integers(1, min(E, 8) + 1))
        logits = np.round(rng.normal(size=E) * 3) / 4
        topk_cases.append({"logits": logits.tolist(), "k": k, "want": mtoy.top_k(logits, k)})
meta["topk"] = topk_cases

# ---------------------------------------------------------------- models
meta["models"] = {}
for name, kw in SPECS.items():
    spec = mconfig.ModelSpec(**kw)
    model = mtoy.build_model(spec)
    hashes = {f: sha(getattr(model, f)) for f in
              ("embed", "attn_q", "attn_k", "attn_v", "attn_o", "router", "expert_in", "expert_out", "head")}
    prompts = [[1, 5, 9, 2], [3], [4, 7], [1, 2, 3, 4, 5, 6, 7, 8]]
    fwd = []
    for pi, prompt in enumerate(prompts):
        little = mtoy.little_forward(model, prompt)
        full = mtoy.full_forward(model, prompt)
        big = mtoy.big_forward(model, prompt, little.router_states)
        bigr = mtoy.big_forward(model, prompt, little.router_states, reuse_gates=True)
        rec = {"prompt": prompt}
        for tag, r in (("little", little), ("full", full), ("big", big), ("big_reuse", bigr)):
            arrays[f"{name}/p{pi}/{tag}/probs"] = r.probs
            arrays[f"{name}/p{pi}/{tag}/states"] = r.router_states
            rec[f"{tag}_selections"] = r.selections
        fwd.append(rec)
    # generate chains
    gens = []
    runs = [dict(gamma=0.7), dict(gamma=0.0), dict(gamma=1.0), dict(gamma=0.5), dict(gamma=0.95)]
    for si in range(4):
        runs.append(dict(gamma=0.95, sampling="Temperature", temperature=2.0, sampling_seed=si))
    runs.append(dict(gamma=0.7, reuse_little_gates=True))
    for ri, pkw in enumerate(runs):
        pol = mconfig.PolicySpec(**pkw)
        prompt = [1 + ri % 7, 2]
        max_len = 16 if name == "c1" else 8
        toks, decs = mtoy.generate(model, prompt, pol, max_len=max_len, record_router_states=True)
        drec = []
        for di, d in enumerate(decs):
            drec.append({"token": d.token, "accepted_by": d.accepted_by, "confidence": d.confidence,
                         "little": d.little_selections, "big": d.big_selections})
            arrays[f"{name}/g{ri}/d{di}/states"] = d.router_states
        gens.append({"policy": pkw, "prompt": prompt, "max_len": max_len, "tokens": toks, "decisions": drec})
    meta["models"][name] = {"spec": kw, "k_little": spec.k_little, "hashes": hashes,
                            "forward": fwd, "generate": gens}

# ---------------------------------------------------------------- policy
sf = []
for probs, g in (([0.9, 0.1], 0.7), ([0.6, 0.4], 0.7), ([0.7, 0.3], 0.7), ([1 / 16] * 16, 0.0),
                 ([0.99, 0.01], 1.0), ([0.5, 0.5], 0.5), ([0.25] * 4, 0.25)):
    sf.append({"probs": probs, "gamma": g, "want": mpolicy.should_fallback(np.array(probs), g)})
meta["should_fallback"] = sf

plans = []
prng = np.random.default_rng(11)
for _ in range(30):
    L = int(prng.integers(1, 8))
    E = int(prng.integers(2, 32))
    k = int(prng.integers(1, E + 1))
    d = int(prng.integers(1, 5))
    states = np.round(prng.normal(size=(L, E)) * 2) / 2
    plan = mpolicy.build_mobile_plan(states, k_big=k, lookahead=d)
    plans.append({"states": states.tolist(), "k": k, "lookahead": d,
                  "targets": [[[x.layer, x.expert] for x in t] for t in plan.targets],
                  "entries": [[e.earliest_issue_layer, e.expert.layer, e.expert.expert, e.after_routing]
                              for e in plan.entries]})
meta["plans"] = plans

meta["injected"] = [{"n": n, "r": r, "flags": mengine.injected_fallback_flags(n, r)}
                    for n, r in ((100, 0.21), (1000, 0.21), (7, 0.0), (7, 1.0), (64, 0.11), (256, 0.11))]

hw = mconfig.load_config_file(mconfig.data_path("rtx4080.json"))["hardware"]
ms = mconfig.load_config_file(mconfig.data_path("olmoe_desk.json"))["model"]
meta["slots_packaged"] = mconfig.hbm_expert_slots(ms, hw)

# ---------------------------------------------------------------- cache traces
traces = []
crng = np.random.default_rng(5)
for ti in range(12):
    slots = int(crng.integers(1, 10))
    t_xfer = float(crng.choice([0.5, 3.0, 100.0]))
    cache = mmemory.HbmCache(slots)
    ch = mmemory.TransferChannel(t_xfer)
    now = 0.0
    ops = []
    for _ in range(300):
        kind = crng.choice(["req", "req", "req", "spec", "pin", "unpin", "token_end", "evict"],
                           p=[0.25, 0.2, 0.1, 0.25, 0.08, 0.06, 0.03, 0.03])
        now += float(crng.uniform(0.0, 2.0))
        key = (int(crng.integers(0, 3)), int(crng.integers(0, 6)))
        eid = mconfig.ExpertId(*key)
        op = {"op": str(kind), "key": list(key), "now": now}
        try:
            if kind in ("req", "spec"):
                r = cache.request(eid, now, ch, speculative=(kind == "spec"))
                op["out"] = None if r is None else [r.status, r.ready_time]
            elif kind == "pin":
                cache.pin(eid)
            elif kind == "unpin":
                cache.unpin(eid)
            elif kind == "token_end":
                cache.token_end()
            else:
                n = int(crng.integers(1, 3))
                op["n"] = n
                use_now = bool(crng.integers(0, 2))
                op["use_now"] = use_now
                v = cache.evict_lru(n, now if use_now else None)
                op["out"] = [[x.layer, x.expert] for x in v]
        except mmemory.CapacityDeadlock:
            op["out"] = "deadlock"
        except ValueError:
            op["out"] = "valueerror"
        op["entries"] = [[x.layer, x.expert] for x in cache.entries()]
        ops.append(op)
    s = cache.stats
    traces.append({"slots": slots, "t_xfer": t_xfer, "ops": ops,
                   "stats": [s.hits, s.coalesced, s.issued, s.evictions, s.deferrals],
                   "transfers": ch.transfers_issued})
meta["cache_traces"] = traces

(OUT / "golden.json").write_text(json.dumps(meta))
np.savez_compressed(OUT / "golden.npz", **arrays)
print(f"wrote {len(arrays)} arrays, json {len(json.dumps(meta)) / 1e3:.0f} kB")
