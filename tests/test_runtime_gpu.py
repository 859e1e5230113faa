"""Graph-captured StepEngine (resident and offloaded experts) vs the oracle's KV decode."""
import numpy as np
import pytest
import torch

from oracle import moe_ref as R
from tests.helpers import DSEEK_MINI, GQA_MINI, QWEN_MINI, QWEN_MINI_NOPE, matched, selections_agree

pytestmark = pytest.mark.gpu


def _oracle(o, prompt, n, flags, full=False):
    dec = R.KVDecoder(o)
    dec.prefill(list(prompt[:-1]))
    toks, out = list(prompt), []
    s = o.spec
    for i in range(n):
        if full:
            probs, states, sel, kv = dec.run([toks[-1]], s.k_big)
            dec.commit(kv)
            out.append((int(np.argmax(probs)), sel, None, states))
        else:
            probs, states, lsel, kv = dec.run([toks[-1]], s.k_little)
            if flags[i]:
                bp, _, bsel, bkv = dec.run([toks[-1]], s.k_big, states)
                dec.commit(bkv)
                out.append((int(np.argmax(bp)), lsel, bsel, states))
            else:
                dec.commit(kv)
                out.append((int(np.argmax(probs)), lsel, None, states))
        toks.append(out[-1][0])
    return out


def _offload_dm(dm, ms):
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.weights import DeviceWeights
    dw = dm.dw
    dw2 = DeviceWeights(ms, dw.device, experts_on_device=False)
    for name in ("embed", "qkv", "o", "router", "shared", "head"):
        setattr(dw2, name, getattr(dw, name))
    dw2.host_experts = dw.experts.cpu().pin_memory()
    return DeviceModel(dw2)


@pytest.mark.parametrize("persistent", [False, True])
@pytest.mark.parametrize("mode", ["resident", "offload"])
@pytest.mark.parametrize("spec_kw", [QWEN_MINI, DSEEK_MINI, QWEN_MINI_NOPE, GQA_MINI])
@pytest.mark.parametrize("full", [False, True])
def test_step_engine_matches_oracle(cuda_ok, mode, spec_kw, full, persistent):
    from paper_2510_12357_b200.offload import OffloadRuntime
    from paper_2510_12357_b200.runtime import StepEngine
    o, ms, dm = matched(spec_kw, "bfloat16")
    rt = None
    if mode == "offload":
        dm = _offload_dm(dm, ms)
        rt = OffloadRuntime(dm.dw, slots=ms.num_experts + 2, lookahead=1)
    eng = StepEngine(dm, 1, 64, runtime=rt, persistent=persistent).build(gamma=0.7)
    assert bool(eng.dp) == persistent
    prompt = [3, 17, 42, 7]
    n = 10
    flags = [bool(i % 3 == 1) for i in range(n)]
    eng.prefill(prompt)
    got = []
    for i in range(n):
        tok, fb = eng.step(forced_fallback=flags[i], full=full)
        lsel = eng.idx["full" if full else "little"][:, 0].cpu().tolist()
        bsel = eng.idx["big"][:, 0].cpu().tolist() if fb else None
        got.append((tok, lsel, bsel))
    want = _oracle(o, prompt, n, flags, full)
    for g, w in zip(got, want):
        assert selections_agree(g[1], w[1], w[3])[0], (g[1], w[1])
        assert (g[2] is None) == (w[2] is None)
        if w[2] is not None:
            assert selections_agree(g[2], w[2], w[3])[0]
    assert [g[0] for g in got] == [w[0] for w in want]
    if rt is not None:
        nbytes, transfers = rt.counters()
        assert transfers == rt.cache.stats.issued


def test_step_engine_confidence_rule(cuda_ok):
    from paper_2510_12357_b200.runtime import StepEngine
    o, ms, dm = matched(QWEN_MINI, "float32")
    for gamma in (0.0, 1.0, 0.05):
        eng = StepEngine(dm, 1, 64).build(gamma=gamma)
        eng.prefill([1, 2, 3])
        for _ in range(6):
            tok, fb = eng.step()
            conf = eng.head["little"]["conf"].item()
            assert fb == (conf <= gamma)


def test_graph_prefill_equals_eager(cuda_ok):
    """A prompt length seen before replays its captured prefill graph (prompt
    ids from a static buffer): KV caches and the following step identical to
    an eager prefill of the same prompt."""
    from paper_2510_12357_b200.runtime import StepEngine
    _, ms, dm = matched(QWEN_MINI, "bfloat16")
    a = StepEngine(dm, 1, 64, persistent=False).build()
    b = StepEngine(dm, 1, 64, persistent=False).build()
    b.prefill_graphs = False
    a.prefill([5, 9, 13, 2, 7, 1])       # eager + capture (length 5)
    a.prefill([3, 17, 42, 8, 11, 4])     # graph replay, other ids
    assert (5, ms.k_big) in a._pf_graphs
    b.prefill([3, 17, 42, 8, 11, 4])     # eager
    torch.cuda.synchronize()
    assert a.sess.pos == b.sess.pos == 5
    assert torch.equal(a.sess.kc[:, :, :, :5], b.sess.kc[:, :, :, :5])
    assert torch.equal(a.sess.vc[:, :, :, :5], b.sess.vc[:, :, :, :5])
    ta, _ = a.step(False, next_token=6)
    tb, _ = b.step(False, next_token=6)
    assert ta == tb and torch.equal(a.states["little"], b.states["little"])
