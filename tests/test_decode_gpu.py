"""KV-cached MoBiLE decode on the GPU vs the oracle's KV restatement.

The KV-cache semantics (accepted pass owns the K/V rows) are an extension the
reference does not pin; parity here is against oracle.generate_kv.
"""
import numpy as np
import pytest
import torch

from oracle import moe_ref as R
from tests.helpers import DSEEK_MINI, QWEN_MINI, matched, selections_agree

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec_kw,dtype", [(QWEN_MINI, "float32"), (QWEN_MINI, "bfloat16"), (DSEEK_MINI, "bfloat16")])
def test_generate_kv_matches_oracle(cuda_ok, spec_kw, dtype):
    from paper_2510_12357_b200 import PolicySpec
    from paper_2510_12357_b200.decode import MobileGenerator
    o, ms, dm = matched(spec_kw, dtype)
    gen = MobileGenerator(dm, max_len=64)
    prompt = [3, 17, 42, 7]
    flags = [bool(i % 3 == 1) for i in range(12)]
    toks, decs = gen.generate(prompt, PolicySpec(gamma=0.7), 12, fallback_flags=flags, stop_at_eos=False)
    # oracle with the same forced flags (no eos stop either)
    o2 = R.OracleWeights(**{**o.__dict__, "spec": R.OracleSpec(**{**spec_kw, "eos_token": -1})}) if False else o
    want_toks, want = _oracle_kv(o, prompt, 12, flags)
    assert [d.accepted_by for d in decs] == [w.accepted_by for w in want]
    for d, w in zip(decs, want):
        ok, _ = selections_agree(d.little_selections, w.little_selections, w.router_states)
        assert ok, (d.little_selections, w.little_selections)
        if w.big_selections is not None:  # replayed: same rule on the little logits
            ok, _ = selections_agree(d.big_selections, w.big_selections, w.router_states)
            assert ok
    assert toks == want_toks


def _oracle_kv(o, prompt, n, flags):
    dec = R.KVDecoder(o)
    dec.prefill(list(prompt[:-1]))
    toks, out = list(prompt), []
    s = o.spec
    for i in range(n):
        probs, states, lsel, kv = dec.run([toks[-1]], s.k_little)
        if flags[i]:
            bp, _, bsel, bkv = dec.run([toks[-1]], s.k_big, states)
            dec.commit(bkv)
            t = int(np.argmax(bp))
            out.append(R.Decision(t, R.ACCEPTED_BIG, float(probs.max()), lsel, bsel, states))
        else:
            dec.commit(kv)
            t = int(np.argmax(probs))
            out.append(R.Decision(t, R.ACCEPTED_LITTLE, float(probs.max()), lsel, None, states))
        toks.append(t)
    return toks, out


def test_confidence_rule_kv(cuda_ok):
    from paper_2510_12357_b200 import PolicySpec
    from paper_2510_12357_b200.decode import MobileGenerator
    o, ms, dm = matched(QWEN_MINI, "float32")
    gen = MobileGenerator(dm, max_len=64)
    for gamma in (0.0, 0.05, 1.0):
        _, decs = gen.generate([1, 2, 3], PolicySpec(gamma=gamma), 10, stop_at_eos=False)
        for d in decs:
            assert (d.accepted_by == "BigFallback") == (d.confidence <= gamma)
        if gamma == 0.0:
            assert all(d.accepted_by == "Little" for d in decs)
        if gamma == 1.0:
            assert all(d.accepted_by == "BigFallback" for d in decs)
