"""`moesim` drop-in alias: `import paper_2510_12357_b200.compat` registers
this package under the reference's module names, so code written against
`moesim` (/root/reference/pkg/src/moesim) runs unchanged on the B200 path:

    moesim            -> paper_2510_12357_b200      (__init__.py re-exports)
    moesim.config     -> .spec      (config.py)
    moesim.toymoe     -> .functional (toymoe.py: build_model, forward, generate ...)
    moesim.policy     -> .policy    (policy.py)
    moesim.memory     -> .memory    (memory.py)
    moesim.engine     -> .sim       (engine.py, incl. selections_from_logits /
                                     fallback_flags_from_confidence /
                                     injected_fallback_flags, engine.py:76-81, 266-277)
    moesim.metrics    -> .metrics   (metrics.py)
    moesim.trace      -> .trace     (trace.py)
    moesim.cli        -> .cli       (cli.py)

The modelled pre-gating competitor (policy.py:119-153) is out of scope
 and is not provided.
"""
from __future__ import annotations

import sys

from . import cli, functional, memory, metrics, policy, sim, spec, trace
import paper_2510_12357_b200 as _pkg

ALIASES = {"moesim": _pkg, "moesim.config": spec, "moesim.toymoe": functional, "moesim.policy": policy,
           "moesim.memory": memory, "moesim.engine": sim, "moesim.metrics": metrics, "moesim.trace": trace,
           "moesim.cli": cli}


def install() -> None:
    for name, mod in ALIASES.items():
        sys.modules.setdefault(name, mod)


install()
