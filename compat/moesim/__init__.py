"""`moesim` on the import path -> this B200 package (paper_2510_12357_b200.compat):
put /root/repo/compat on PYTHONPATH and reference code -- `import moesim`,
`from moesim.toymoe import generate`, `python -m moesim ...` -- runs unchanged
on the sm_100a kernels.  (Only for drop-in use; never on the path together
with the reference package itself.)"""
import sys

import paper_2510_12357_b200.compat as _compat

sys.modules[__name__] = _compat.ALIASES["moesim"]
