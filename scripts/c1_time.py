"""C1 drop-in generate timing: libmobile _lin vs the torch matmul it replaced (experiment)."""
import sys
import time
from pathlib import Path

import torch
import torch.nn.functional as Fn

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2510_12357_b200 as M  # noqa: E402
from paper_2510_12357_b200.model import DeviceModel  # noqa: E402

kw = dict(num_layers=2, num_experts=16, k_big=4, k_little=2, hidden_dim=256, vocab_size=256, seed=0)
prompt = [3, 17, 42, 5]
om = M.build_model(M.ModelSpec(**kw))


def run(tag):
    M.generate(om, prompt, M.PolicySpec(), 2)
    torch.cuda.synchronize()
    for rep in range(2):
        w0 = time.perf_counter()
        toks, dec = M.generate(om, prompt, M.PolicySpec(), 24)
        torch.cuda.synchronize()
        print(tag, rep, round(24 / (time.perf_counter() - w0), 1), "tok/s", flush=True)


run("libmobile_lin")
orig = DeviceModel._lin


def torch_lin(self, h, w, resid=None):
    w = self.dw.plain(w)
    y = Fn.linear(h, w) if w.dtype == torch.float32 else Fn.linear(h.to(w.dtype), w).to(torch.float32)
    return y if resid is None else resid + y


DeviceModel._lin = torch_lin
run("torch_lin")
