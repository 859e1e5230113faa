"""Pin the CPU oracle (oracle/moe_ref.py) to the reference's golden vectors.

The golden vectors were produced by the unmodified reference (`moesim`) via
tests/golden/make_golden.py; these tests run anywhere (no GPU, no reference).
"""
import hashlib

import numpy as np
import pytest

from oracle import moe_ref as R


def _spec(kw):
    return R.OracleSpec(**kw)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_topk_matches_reference(golden):
    meta, _ = golden
    for case in meta["topk"]:
        logits = np.array(case["logits"])
        assert R.top_k(logits, case["k"]) == case["want"]
        assert R.reference_top_k(list(logits), case["k"]) == case["want"] or any(
            x == 0.0 for x in logits)  # python sort keeps -0.0 == 0.0 too


def test_topk_errors():
    with pytest.raises(ValueError, match="exceeds"):
        R.top_k(np.zeros(4), 5)
    with pytest.raises(ValueError, match="finite"):
        R.top_k(np.array([1.0, np.nan]), 1)


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_weights_bit_identical(golden, name):
    meta, _ = golden
    m = meta["models"][name]
    W = R.build_weights(_spec(m["spec"]))
    for field, h in m["hashes"].items():
        assert _sha(getattr(W, field)) == h, field


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_forward_bit_identical(golden, name):
    meta, arrays = golden
    m = meta["models"][name]
    spec = _spec(m["spec"])
    W = R.build_weights(spec)
    for pi, rec in enumerate(m["forward"]):
        prompt = rec["prompt"]
        little = R.forward(W, prompt, spec.k_little)
        full = R.forward(W, prompt, spec.k_big)
        big = R.forward(W, prompt, spec.k_big, little.router_states)
        bigr = R.forward(W, prompt, spec.k_big, little.router_states, reuse_gates=True)
        for tag, r in (("little", little), ("full", full), ("big", big), ("big_reuse", bigr)):
            assert np.array_equal(r.probs, arrays[f"{name}/p{pi}/{tag}/probs"]), (tag, pi)
            assert np.array_equal(r.router_states, arrays[f"{name}/p{pi}/{tag}/states"]), (tag, pi)
            assert r.selections == rec[f"{tag}_selections"], (tag, pi)


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_generate_identical(golden, name):
    meta, arrays = golden
    m = meta["models"][name]
    spec = _spec(m["spec"])
    W = R.build_weights(spec)
    for gi, g in enumerate(m["generate"]):
        p = dict(g["policy"])
        toks, decs = R.generate(W, g["prompt"], p.get("gamma", 0.7), g["max_len"],
                                sampling=p.get("sampling", "Greedy"), temperature=p.get("temperature", 1.0),
                                sampling_seed=p.get("sampling_seed", 0),
                                reuse_gates=p.get("reuse_little_gates", False), record_router_states=True)
        assert toks == g["tokens"]
        for di, (d, want) in enumerate(zip(decs, g["decisions"])):
            assert d.token == want["token"] and d.accepted_by == want["accepted_by"]
            assert d.confidence == want["confidence"]
            assert d.little_selections == want["little"]
            assert d.big_selections == want["big"]
            assert np.array_equal(d.router_states, arrays[f"{name}/g{gi}/d{di}/states"])


def test_should_fallback(golden):
    meta, _ = golden
    for c in meta["should_fallback"]:
        assert R.should_fallback(np.array(c["probs"]), c["gamma"]) == c["want"]
    with pytest.raises(ValueError, match="sums to"):
        R.should_fallback(np.array([0.5, 0.2]), 0.7)


def test_plans(golden):
    meta, _ = golden
    for c in meta["plans"]:
        targets, entries = R.build_mobile_plan(np.array(c["states"]), c["k"], c["lookahead"])
        assert [[list(t) for t in row] for row in targets] == c["targets"]
        assert [list(e) for e in entries] == c["entries"]


def test_injected_flags(golden):
    meta, _ = golden
    for c in meta["injected"]:
        assert R.injected_fallback_flags(c["n"], c["r"]) == c["flags"]


def test_slots_formula(golden):
    meta, _ = golden
    # olmoe_desk.json + rtx4080.json: L16, dense 8MiB, 16GiB cap, 6GiB reserved, 64MiB experts
    assert R.hbm_expert_slots(16, 8 * 2**20, 16 * 2**30, 6 * 2**30, 64 * 2**20, 8) == meta["slots_packaged"]


def test_cache_traces(golden):
    meta, _ = golden
    for tr in meta["cache_traces"]:
        cache, ch = R.CacheRef(tr["slots"]), R.ChannelRef(tr["t_xfer"])
        for op in tr["ops"]:
            key = tuple(op["key"])
            k = op["op"]
            try:
                if k in ("req", "spec"):
                    r = cache.request(key, op["now"], ch, speculative=(k == "spec"))
                    assert (None if r is None else [r[0], r[1]]) == op["out"]
                elif k == "pin":
                    cache.pin(key)
                elif k == "unpin":
                    cache.unpin(key)
                elif k == "token_end":
                    cache.token_end()
                else:
                    v = cache.evict_lru(op["n"], op["now"] if op["use_now"] else None)
                    assert [list(x) for x in v] == op["out"]
            except R.CapacityDeadlockRef:
                assert op["out"] == "deadlock"
            except ValueError:
                assert op["out"] == "valueerror"
            assert [list(x) for x in cache.ready] == op["entries"]
        assert [cache.hits, cache.coalesced, cache.issued, cache.evictions, cache.deferrals] == tr["stats"]
        assert ch.transfers_issued == tr["transfers"]


def test_kv_decode_first_step_equals_recompute():
    """KV decode restatement: with a 1-token prompt the first little step is the
    recompute forward (no earlier positions exist)."""
    spec = R.OracleSpec(num_layers=2, num_experts=8, k_big=4, hidden_dim=16, vocab_size=32, seed=3)
    W = R.build_weights(spec)
    dec = R.KVDecoder(W)
    probs, states, sels, _ = dec.run([5], spec.k_little)
    ref = R.forward(W, [5], spec.k_little)
    np.testing.assert_allclose(probs, ref.probs, rtol=1e-12)
    assert sels == ref.selections


def test_kv_decode_full_width_equals_recompute():
    """At k_little == k_big with no fallback dependence, KV decode == recompute."""
    spec = R.OracleSpec(num_layers=2, num_experts=8, k_big=4, k_little=4, hidden_dim=16, vocab_size=32, seed=3)
    W = R.build_weights(spec)
    toks_kv, _ = R.generate_kv(W, [1, 2, 3], 0.7, 6)
    toks_rc, _ = R.generate(W, [1, 2, 3], 0.7, 6)
    assert toks_kv == toks_rc
