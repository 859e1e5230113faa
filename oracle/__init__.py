"""CPU oracle for the MoBiLE MoE hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import anything under `oracle/`, and only as the
checker or the timed CPU reference -- never as the product path.  The product
package `paper_2510_12357_b200` must never import this package.

`moe_ref` is a NumPy restatement of the reference's functional path
(`/root/reference/pkg/src/moesim/toymoe.py`, `policy.py`, `memory.py`,
`engine.py:266-277`), generalised to the real-shape extensions the build adds
(SwiGLU experts, shared experts, HF-style gating, multi-head attention, a
KV-cache decode mode).  Its toy-setting behaviour is pinned against golden
vectors generated from the importable reference (`tests/golden/make_golden.py`):
bit-identical fp64 for forward/generate, identical plans and cache traces.
The real-shape extensions are "parity unpinned" by the reference (it has no
SwiGLU/shared/KV-cache counterpart) and are anchored to this restatement only.
"""
