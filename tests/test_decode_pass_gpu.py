"""Persistent decode-pass kernel (decode_pass.cu) vs the oracle and vs the
per-op kernel engine on identical weights."""
from dataclasses import replace

import numpy as np
import pytest
import torch

from tests.helpers import GQA_MINI, OLMOE_MINI, QWEN_MINI, matched, selections_agree
from tests.test_runtime_gpu import _oracle

pytestmark = pytest.mark.gpu

TOY = dict(num_layers=2, num_experts=16, k_big=4, k_little=2, hidden_dim=256, vocab_size=256, seed=0)


@pytest.mark.parametrize("spec_kw,dtype", [(TOY, "float32"), (OLMOE_MINI, "bfloat16"), (QWEN_MINI, "float32"),
                                           (GQA_MINI, "bfloat16")])
@pytest.mark.parametrize("full", [False, True])
def test_persistent_matches_oracle(cuda_ok, spec_kw, dtype, full):
    from paper_2510_12357_b200.runtime import StepEngine
    o, ms, dm = matched(spec_kw, dtype)
    eng = StepEngine(dm, 1, 64, persistent=True).build(gamma=0.7)
    prompt = [3, 17, 42, 7, 9]
    n = 12
    flags = [bool(i % 3 == 1) for i in range(n)]
    eng.prefill(prompt)
    got = []
    for i in range(n):
        tok, fb = eng.step(forced_fallback=flags[i], full=full)
        lsel = eng.idx["full" if full else "little"][:, 0].cpu().tolist()
        bsel = eng.idx["big"][:, 0].cpu().tolist() if fb else None
        got.append((tok, lsel, bsel, eng.states["full" if full else "little"][:, 0].cpu().numpy()))
    want = _oracle(o, prompt, n, flags, full)
    assert int(eng.dp_flags.item()) == 0
    for g, w in zip(got, want):
        assert selections_agree(g[1], w[1], w[3])[0], (g[1], w[1])
        if w[2] is not None:
            assert selections_agree(g[2], w[2], w[3])[0]
        err = np.abs(g[3] - w[3]).max() / np.abs(w[3]).max()
        assert err < (1e-4 if dtype == "float32" else 2e-2), err
    assert [g[0] for g in got] == [w[0] for w in want]


@pytest.mark.parametrize("preset", ["c2", "c3", "c4"])
def test_persistent_equals_per_op_real_shape(cuda_ok, preset):
    """Real widths (d=2048, 60-64 experts, shared experts), 3 layers: the
    persistent pass and the per-op engine agree on every selection and token."""
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    spec = replace(PRESETS[preset], num_layers=3)
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=3))
    a = StepEngine(dm, 1, 96, persistent=True).build()
    b = StepEngine(dm, 1, 96, persistent=False).build()
    prompt = np.random.default_rng(0).integers(1, spec.vocab_size, size=40).tolist()
    stream = np.random.default_rng(1).integers(1, spec.vocab_size, size=16).tolist()
    a.prefill(prompt)
    b.prefill(prompt)
    for i in range(12):
        fb = i % 4 == 2
        for e in (a, b):
            e.step(forced_fallback=fb, next_token=stream[i])
        for kd in ("little", "big") if fb else ("little",):
            sa, sb = a.states[kd].cpu().numpy(), b.states[kd].cpu().numpy()
            assert np.abs(sa - sb).max() <= 1e-3 * np.abs(sb).max()
            ia, ib = a.idx[kd].cpu().tolist(), b.idx[kd].cpu().tolist()
            for l in range(spec.num_layers):
                assert selections_agree([ia[l][0]], [ib[l][0]], sb[l:l + 1, 0], tol=1e-4)[0]
        ca, cb = a.head["little"]["conf"].item(), b.head["little"]["conf"].item()
        assert abs(ca - cb) <= 1e-3 * max(cb, 1e-6)
        assert a.head["little"]["argmax"].item() == b.head["little"]["argmax"].item()
    assert int(a.dp_flags.item()) == 0


@pytest.mark.parametrize("slots", [6, 14])
def test_zero_sync_offload_equals_segmented(cuda_ok, slots):
    """One-launch zero-sync offloaded passes vs the segmented driver: same
    tokens, selections, cache decisions (hits / issued / coalesced) and
    transfers (engine.py:121-169 protocol either way)."""
    from paper_2510_12357_b200.offload import OffloadRuntime
    from paper_2510_12357_b200.runtime import StepEngine
    from tests.test_runtime_gpu import _offload_dm
    o, ms, dm0 = matched(QWEN_MINI, "bfloat16")
    res = []
    for zs in (False, True):
        dm = _offload_dm(dm0, ms)
        rt = OffloadRuntime(dm.dw, slots=slots, lookahead=1)
        eng = StepEngine(dm, 1, 64, runtime=rt, persistent=True, zero_sync=zs).build(gamma=0.7)
        eng.prefill([3, 17, 42, 7])
        toks, sels = [], []
        for i in range(12):
            tok, fb = eng.step(forced_fallback=(i % 3 == 1), full=(i % 5 == 4))
            toks.append(tok)
            sels.append(eng.idx["little"][:, 0].cpu().tolist())
        st = rt.cache.stats
        res.append((toks, sels, (st.hits, st.issued, st.coalesced), rt.counters()))
        assert int(eng.dp_flags.item()) == 0
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    assert res[0][2] == res[1][2]
    assert res[0][3] == res[1][3]


@pytest.mark.parametrize("preset,B", [("c4", 2), ("c4", 4), ("c3", 3), ("c5", 1)])
def test_persistent_batched_and_wide_equal_per_op(cuda_ok, preset, B):
    """Batched decode (B = 2..4 sequences, the TT = 2 / 4 kernels) and the
    Mixtral width (d = 4096, 2-stage ring): one pass of every kind from the
    same random KV state, persistent kernel vs per-op engine."""
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    spec = replace(PRESETS[preset], num_layers=2)
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=4))
    ctx = 37
    engines = [StepEngine(dm, B, 64, persistent=p, gemm=False).build() for p in (True, False)]
    g = torch.Generator(device="cuda").manual_seed(0)
    kc = torch.randn(engines[0].sess.kc.shape, device="cuda", generator=g)
    vc = torch.randn(engines[0].sess.vc.shape, device="cuda", generator=g)
    tok = torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32, generator=g)
    for kd in ("little", "big", "full"):
        for e in engines:
            e.sess.kc.copy_(kc)
            e.sess.vc.copy_(vc)
            e.pos.fill_(ctx)
            e.tok.copy_(tok)
            if kd == "big":  # replay the same little logits in both
                e.states["little"].copy_(engines[1].states["little"])
            torch.cuda.synchronize()  # state set on the default stream; passes run on the engine's stream
            e.run_pass(kd)
        torch.cuda.synchronize()
        a, b = engines
        sa, sb = a.states[kd].cpu().numpy(), b.states[kd].cpu().numpy()
        assert np.abs(sa - sb).max() <= 1e-3 * np.abs(sb).max(), (kd, np.abs(sa - sb).max(axis=-1))
        ia, ib = a.idx[kd].cpu().numpy(), b.idx[kd].cpu().numpy()
        for l in range(spec.num_layers):
            for s in range(B):
                assert selections_agree([ia[l, s].tolist()], [ib[l, s].tolist()], sb[l:l + 1, s], tol=1e-4)[0]
        ca, cb = a.head[kd]["conf"].cpu().numpy(), b.head[kd]["conf"].cpu().numpy()
        assert np.abs(ca - cb).max() <= 1e-3 * max(np.abs(cb).max(), 1e-6), kd
        assert (a.head[kd]["argmax"].cpu() == b.head[kd]["argmax"].cpu()).all(), kd
        # the new position's K/V rows went to the same cache slots
        assert torch.allclose(a.sess.kc[:, :, :, ctx], b.sess.kc[:, :, :, ctx], rtol=1e-3, atol=1e-3)
    assert int(engines[0].dp_flags.item()) == 0


@pytest.mark.parametrize("preset,B", [("c4", 6), ("c3", 130)])
def test_large_batch_gemm_path_equals_batch1(cuda_ok, preset, B):
    """Large-batch decode (B > 4): QKV / O / head on the tcgen05 GEMM (bf16
    operands) and the experts on the grouped GEMM, vs batch-1 engines on the
    same sequences (GEMV path, f32 activations).  Tolerance: bf16 rounding of
    the GEMM activations (2e-2 of the row's largest logit); selections may
    differ only inside that tolerance; the head's argmax must be a maximiser
    of the batch-1 logits within it."""
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    spec = replace(PRESETS[preset], num_layers=2)
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=5))
    ctx = 29
    big = StepEngine(dm, B, 48).build()
    assert big.gemm_path and not big.dp
    one = StepEngine(dm, 1, 48, persistent=False).build()
    g = torch.Generator(device="cuda").manual_seed(1)
    big.sess.kc.copy_(torch.randn(big.sess.kc.shape, device="cuda", generator=g))
    big.sess.vc.copy_(torch.randn(big.sess.vc.shape, device="cuda", generator=g))
    big.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32, generator=g))
    big.pos.fill_(ctx)
    kc0, vc0 = big.sess.kc.clone(), big.sess.vc.clone()
    rows = sorted({0, B // 2, B - 1})
    tol = 2e-2
    for kd in ("little", "full"):
        big.sess.kc.copy_(kc0)
        big.sess.vc.copy_(vc0)
        torch.cuda.synchronize()
        big.run_pass(kd)
        torch.cuda.synchronize()
        for s_ in rows:
            one.sess.kc.copy_(kc0[:, s_:s_ + 1])
            one.sess.vc.copy_(vc0[:, s_:s_ + 1])
            one.pos.fill_(ctx)
            one.tok.copy_(big.tok[s_:s_ + 1])
            torch.cuda.synchronize()
            one.run_pass(kd)
            torch.cuda.synchronize()
            sa, sb = big.states[kd][:, s_].cpu().numpy(), one.states[kd][:, 0].cpu().numpy()
            assert np.abs(sa - sb).max() <= tol * np.abs(sb).max(), (kd, s_)
            ia, ib = big.idx[kd][:, s_].cpu().tolist(), one.idx[kd][:, 0].cpu().tolist()
            assert selections_agree(ia, ib, sb, tol=tol)[0], (kd, s_, ia, ib)
            # final LN(x) at bf16 tolerance; the head (GEMM on bf16(LN x) +
            # row confidence) exactly against torch on the same operand
            la, lb = big.ln[s_].double(), one.ln[0].double()
            assert float((la - lb).abs().max()) <= tol * float(lb.abs().max()), (kd, s_)
            ref = (la.to(torch.bfloat16).double() @ dm.dw.head.double().T) * spec.logit_scale
            conf = float(torch.softmax(ref, dim=0).max())
            ca = float(big.head[kd]["conf"][s_])
            assert abs(ca - conf) <= 1e-3 * conf + 1e-6, (kd, s_, ca, conf)
            am = int(big.head[kd]["argmax"][s_])
            assert float(ref.max() - ref[am]) <= 1e-5 * float(ref.abs().max()), (kd, s_)
            assert bool(big.head[kd]["fallback"][s_]) == (ca <= 0.7)
            assert torch.allclose(big.sess.kc[:, s_, :, ctx], one.sess.kc[:, 0, :, ctx], rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("B", [8, 64])
def test_shared_fork_bit_identical(cuda_ok, monkeypatch, B):
    """Batched GEMM path: the shared experts forked onto a side stream (from
    the residual, LN in the gather) give the same pass, bit for bit, as the
    serial order (shared experts after routing, from the router's h2) -- in
    graph replay, for little and full passes."""
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    spec = replace(PRESETS["c4"], num_layers=3)
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=9))
    engines = []
    for fork in ("1", "0"):
        monkeypatch.setenv("MOBILE_SHARED_FORK", fork)
        e = StepEngine(dm, B, 40).build()
        assert e.gemm_path and e.fork_shared == (fork == "1")
        g = torch.Generator(device="cuda").manual_seed(3)
        e.sess.kc.copy_(torch.randn(e.sess.kc.shape, device="cuda", generator=g))
        e.sess.vc.copy_(torch.randn(e.sess.vc.shape, device="cuda", generator=g))
        e.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32, generator=g))
        e.pos.fill_(21)
        engines.append(e)
    for kd in ("little", "full"):
        outs = []
        for e in engines:
            torch.cuda.synchronize()
            e.graphs[kd].replay()
            torch.cuda.synchronize()
            outs.append((e.states[kd].clone(), e.idx[kd].clone(), e.ln.clone(), e.head[kd]["conf"].clone()))
        for a, b in zip(*outs):
            assert torch.equal(a, b), kd


@pytest.mark.parametrize("B", [1, 2, 4])
def test_forced_gemm_path_small_batch_with_shared_experts(cuda_ok, B):
    """StepEngine(gemm=True) below TC_MIN_TOKENS on a model with shared
    experts: the experts stream on the GEMV engine, so no shared-expert fork
    may be left unjoined (graph capture used to fail with 'capturing stream
    has unjoined work'); the passes agree with the per-op engine within the
    GEMM path's bf16 tolerance."""
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    spec = replace(PRESETS["c4"], num_layers=2)
    dm = DeviceModel(DeviceWeights.random(spec, torch.device("cuda"), seed=7))
    gem = StepEngine(dm, B, 48, gemm=True).build()
    ref = StepEngine(dm, B, 48, gemm=False, persistent=False).build()
    assert gem.gemm_path and not gem.fork_shared
    g = torch.Generator(device="cuda").manual_seed(2)
    kc = torch.randn(gem.sess.kc.shape, device="cuda", generator=g)
    vc = torch.randn(gem.sess.vc.shape, device="cuda", generator=g)
    tok = torch.randint(1, spec.vocab_size, (B,), device="cuda", dtype=torch.int32, generator=g)
    for e in (gem, ref):
        e.sess.kc.copy_(kc)
        e.sess.vc.copy_(vc)
        e.tok.copy_(tok)
        e.pos.fill_(20)
        e.run_pass("little")
        e.stream.synchronize()
    a, b = gem.states["little"].float(), ref.states["little"].float()
    assert torch.isfinite(a).all()
    assert (a - b).abs().max().item() <= 2e-2 * b.abs().max().item()
