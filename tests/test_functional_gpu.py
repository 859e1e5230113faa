"""Drop-in API (`forward`, `generate`, ...) on the GPU vs the reference's golden vectors.

Bar: selections and fallback decisions identical; probabilities / router logits
within fp32 rel 1e-4 of the reference's fp64 values.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _model(meta, name):
    import paper_2510_12357_b200 as M
    m = meta["models"][name]
    return M.build_model(M.ModelSpec(**m["spec"])), m


def _close(a, b, rtol=1e-4):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b))) < rtol


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_weights_match_reference(golden, name, cuda_ok):
    import hashlib
    meta, _ = golden
    model, m = _model(meta, name)
    for f, h in m["hashes"].items():
        assert hashlib.sha256(np.ascontiguousarray(getattr(model, f)).tobytes()).hexdigest() == h


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_forward_matches_golden(golden, name, cuda_ok):
    import paper_2510_12357_b200 as M
    meta, arrays = golden
    model, m = _model(meta, name)
    for pi, rec in enumerate(m["forward"]):
        prompt = rec["prompt"]
        little = M.little_forward(model, prompt)
        full = M.full_forward(model, prompt)
        big = M.big_forward(model, prompt, arrays[f"{name}/p{pi}/little/states"])
        bigr = M.big_forward(model, prompt, arrays[f"{name}/p{pi}/little/states"], reuse_gates=True)
        for tag, r in (("little", little), ("full", full), ("big", big), ("big_reuse", bigr)):
            assert r.selections == rec[f"{tag}_selections"], (name, pi, tag)
            assert _close(r.probs, arrays[f"{name}/p{pi}/{tag}/probs"]), (name, pi, tag)
            assert _close(r.router_states, arrays[f"{name}/p{pi}/{tag}/states"]), (name, pi, tag)
            assert abs(r.probs.sum() - 1.0) < 1e-9


@pytest.mark.parametrize("name", ["small", "c1", "a7"])
def test_generate_matches_golden(golden, name, cuda_ok):
    import paper_2510_12357_b200 as M
    meta, arrays = golden
    model, m = _model(meta, name)
    for gi, g in enumerate(m["generate"]):
        pol = M.PolicySpec(**g["policy"])
        toks, decs = M.generate(model, g["prompt"], pol, max_len=g["max_len"], record_router_states=True)
        assert toks == g["tokens"], (name, gi)
        for di, (d, want) in enumerate(zip(decs, g["decisions"])):
            assert d.accepted_by == want["accepted_by"]
            assert abs(d.confidence - want["confidence"]) < 1e-4 * want["confidence"]
            assert d.little_selections == want["little"]
            assert d.big_selections == want["big"]
            assert _close(d.router_states, arrays[f"{name}/g{gi}/d{di}/states"])


# ---- reference behaviour (restated from the reference's own test intents) ----
SMALL = dict(num_layers=3, num_experts=8, k_big=4, k_little=2, hidden_dim=16, vocab_size=32, seed=7)


@pytest.fixture(scope="module")
def small(cuda_ok):
    import paper_2510_12357_b200 as M
    return M.build_model(M.ModelSpec(**SMALL))


def test_topk_api(cuda_ok):
    import paper_2510_12357_b200 as M
    assert M.top_k(np.array([0.5, 2.0, 1.0, 3.0]), 2) == [3, 1]
    assert M.top_k(np.array([5.0, 5.0, 5.0]), 2) == [0, 1]
    with pytest.raises(ValueError, match="exceeds"):
        M.top_k(np.zeros(4), 5)
    with pytest.raises(ValueError, match="finite"):
        M.top_k(np.array([1.0, np.nan]), 1)


def test_softmax_api(cuda_ok):
    import paper_2510_12357_b200 as M
    p = M.softmax(np.array([1.0, 2.0, 3.0]))
    assert abs(p.sum() - 1.0) < 1e-12 and np.all(p > 0)
    assert np.allclose(M.softmax(np.array([0.3, -1.2, 2.0])), M.softmax(np.array([100.3, 98.8, 102.0])))


def test_little_equals_full_bitwise_when_widths_match(cuda_ok):
    import paper_2510_12357_b200 as M
    model = M.build_model(M.ModelSpec(**{**SMALL, "k_little": 4, "seed": 11}))
    rng = np.random.default_rng(0)
    for _ in range(10):
        prompt = [int(t) for t in rng.integers(1, 32, size=int(rng.integers(2, 7)))]
        a, b = M.little_forward(model, prompt), M.full_forward(model, prompt)
        assert np.array_equal(a.probs, b.probs) and a.selections == b.selections


def test_replay_and_subset(small):
    import paper_2510_12357_b200 as M
    from oracle.moe_ref import reference_top_k
    toks = [1, 5, 9, 2]
    little = M.little_forward(small, toks)
    big = M.big_forward(small, toks, little.router_states)
    for layer in range(3):
        assert big.selections[layer] == reference_top_k(list(little.router_states[layer]), 4)
        assert set(little.selections[layer]) <= set(big.selections[layer])
    fresh = M.big_forward(small, toks, little.router_states, reuse_gates=False)
    reused = M.big_forward(small, toks, little.router_states, reuse_gates=True)
    assert fresh.selections == reused.selections


def test_errors(small):
    import paper_2510_12357_b200 as M
    with pytest.raises(ValueError, match="empty"):
        M.little_forward(small, [])
    with pytest.raises(ValueError, match="vocab"):
        M.little_forward(small, [99])
    with pytest.raises(ValueError, match="shape"):
        M.forward(small, [1, 2], 4, replay_states=np.zeros((2, 8)))
    with pytest.raises(ValueError, match="prompt"):
        M.generate(small, [], M.PolicySpec(), max_len=4)
    with pytest.raises(ValueError, match="max_len"):
        M.generate(small, [1], M.PolicySpec(), max_len=0)
    with pytest.raises(M.ConfigError, match="hidden_dim"):
        M.build_model(M.ModelSpec(num_layers=1, num_experts=4, k_big=2, hidden_dim=4096))


def test_gamma_extremes_and_strict_rule(small):
    import paper_2510_12357_b200 as M
    _, acc = M.generate(small, [1, 2], M.PolicySpec(gamma=0.0), max_len=6)
    assert all(d.accepted_by == M.ACCEPTED_LITTLE for d in acc)
    _, rej = M.generate(small, [1, 2], M.PolicySpec(gamma=1.0), max_len=6)
    assert all(d.accepted_by == M.ACCEPTED_BIG and d.router_states is not None for d in rej)
    _, mix = M.generate(small, [3, 1], M.PolicySpec(gamma=0.6), max_len=12)
    assert all((d.accepted_by == M.ACCEPTED_BIG) == (d.confidence <= 0.6) for d in mix)


def test_should_fallback_api(golden, cuda_ok):
    import paper_2510_12357_b200 as M
    meta, _ = golden
    for c in meta["should_fallback"]:
        assert M.should_fallback(np.array(c["probs"]), c["gamma"]) == c["want"]
    with pytest.raises(ValueError, match="sums to"):
        M.should_fallback(np.array([0.5, 0.2]), 0.7)


def test_build_mobile_plan_golden(golden, cuda_ok):
    import paper_2510_12357_b200 as M
    meta, _ = golden
    for c in meta["plans"]:
        plan = M.build_mobile_plan(np.array(c["states"]), c["k"], c["lookahead"])
        assert [[[x.layer, x.expert] for x in t] for t in plan.targets] == c["targets"]
        assert [[e.earliest_issue_layer, e.expert.layer, e.expert.expert, e.after_routing] for e in plan.entries] == c["entries"]
    with pytest.raises(ValueError, match="lookahead"):
        M.build_mobile_plan(np.zeros((2, 4)), 2, 0)
    with pytest.raises(ValueError, match="2-D"):
        M.build_mobile_plan(np.zeros(4), 2, 1)
