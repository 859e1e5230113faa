"""Benchmark: decode tokens/s, MoBiLE vs the full-top-k offload baseline,
Qwen1.5-MoE-A2.7B shape (BASELINE.json metric; configs[2] = C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (C3): Qwen1.5-MoE-A2.7B shape (d2048, 24 layers, 60 routed experts
top-4 / little top-2, one 5632-wide sigmoid-gated shared expert, V151936),
random-init bf16 weights.  Routed experts live in pinned host DRAM; the HBM
expert cache is capped by the reference's own budget formula
(hbm_expert_slots, config.py:204-218) at the paper's 16 GiB / 6 GiB-reserved
consumer setting (rtx4080.json) -> 477 slots of 1440 experts.  Batch-1 greedy
decode after a 512-token prompt; the fallback ratio is pinned at the paper's
Qwen r = 0.11 with engine.injected_fallback_flags.  A step is
one decoded token.  Every token streams ~4.7 GB of weights (>> 126 MB L2), so
no L2 flush is needed between steps.

The full-top-k baseline (every token at k=4, experts loaded on demand, the
reference's simulate_full_stream) runs on the same stack in the same process;
its tokens/s and the MoBiLE/full speed-up are reported beside `value`.

`--impl reference` times the reference's CPU path of the same decode (the
oracle's NumPy restatement in fp32 on the host cores; the reference package
cannot build d=2048 models) and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s, MoBiLE vs full-top-k offload baseline, Qwen1.5-MoE-A2.7B"
WORKLOAD = ("C3: Qwen1.5-MoE-A2.7B shape, experts in pinned host DRAM, capped HBM expert cache "
            "(477 slots = hbm_expert_slots at 16 GiB cap / 6 GiB reserved), batch-1 greedy decode, "
            "prompt 512, injected fallback ratio r=0.11")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--r", type=float, default=0.11)
    ap.add_argument("--cap-gib", type=float, default=16.0)
    ap.add_argument("--reserved-gib", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=0, help="CPU-baseline tokens (default: --steps)")
    ap.add_argument("--layers", type=int, default=0, help="debug only: fewer layers (invalidates the number)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config (C2/C4/C5) block")
    ap.add_argument("--no-ep", action="store_true", help="skip the expert-parallel (C4 batched) block")
    ap.add_argument("--ep-batch", type=int, default=64, help="sequences per rank in the expert-parallel block")
    ap.add_argument("--configs", default="c1,c2,c4,c5", help="configs of the per-config block")
    return ap.parse_args()


# ----------------------------------------------------------------------------- dist
def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if os.environ.get("MOBILE_BENCH_SHARE_GPU") == "1":
            # functional test of the multi-rank path on a 1-GPU box: every rank on
            # cuda:0 (the EP mailboxes map through CUDA IPC), gloo for the host
            # collectives (NCCL refuses two ranks on one GPU); numbers meaningless
            backend, local = "gloo", 0
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v: float, device=None) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML in a
    20 ms polling thread (the timed region of the headline is ~0.2 s, too short
    for nvidia-smi's own start-up + 200 ms period), nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

            def sample():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), [self.NAMES[i] for i, b in enumerate(bits) if rs & b]))

            def poll():
                while True:
                    sample()
                    if self.stop.wait(0.01):
                        break
            self.sample = sample
            # the timed loop is Python calling into ctypes: a short GIL switch
            # interval lets the polling thread run every ~10 ms
            self.switch = sys.getswitchinterval()
            sys.setswitchinterval(0.001)
            self.nvml = N
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if r[0].replace(".", "").isdigit() and r[1].replace(".", "").isdigit():
                self.rows.append((float(r[0]), float(r[1]), [self.NAMES[i] for i in range(4)
                                                             if len(r) > 3 + i and "Active" in r[3 + i]
                                                             and "Not" not in r[3 + i]]))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
            sys.setswitchinterval(self.switch)
            try:
                self.sample()  # the clock at the end of the timed region
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        import statistics
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d.get("decode_pass_dram_bytes_per_launch")
    except Exception:
        return None


def bench_config(args, ws, slots, routed_experts, layers):
    """The workload's config block -- identical for both arms (same_config)."""
    return {"workload": WORKLOAD, "model": "Qwen1.5-MoE-A2.7B-shape", "global_batch": ws,
            "seq_len": args.prompt_len + args.warmup + args.steps, "context": args.prompt_len,
            "parallelism": f"replicas{ws}" if ws > 1 else "single", "hbm_expert_slots": slots,
            "routed_experts": routed_experts, "r_injected": args.r, "lookahead": 2, "gamma": 0.7,
            "l2": "inputs > L2: ~4.7 GB of weights streamed per token (no flush)", "layers": layers}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    from paper_2510_12357_b200 import PolicySpec, hbm_expert_slots
    from paper_2510_12357_b200 import kernels as K
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.offload import OffloadRuntime
    from paper_2510_12357_b200.policy import injected_fallback_flags
    from paper_2510_12357_b200.presets import QWEN15_MOE, with_byte_sizes
    from paper_2510_12357_b200.spec import HardwareSpec
    from paper_2510_12357_b200.weights import DeviceWeights
    from dataclasses import replace

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    spec = QWEN15_MOE if not args.layers else replace(QWEN15_MOE, num_layers=args.layers)
    spec = with_byte_sizes(spec)
    hw = HardwareSpec(hbm_capacity=int(args.cap_gib * 2**30), reserved=int(args.reserved_gib * 2**30))
    slots = hbm_expert_slots(spec, hw)
    t0 = time.time()
    dw = DeviceWeights.random(spec, dev, seed=rank, experts_on_device=False)
    t_init = time.time() - t0
    dm = DeviceModel(dw)
    prompt = np.random.default_rng(1 + rank).integers(1, spec.vocab_size, size=args.prompt_len).tolist()
    K_, W_ = args.steps, args.warmup
    flags = injected_fallback_flags(W_ + K_, args.r)
    policy = PolicySpec(gamma=0.7)
    max_len = args.prompt_len + W_ + K_ + 8

    # synthetic input stream: the step inputs are teacher-forced random ids so
    # routing varies token to token as in real text (greedy feedback on random
    # weights collapses onto one repeated token and a 100%-hit cache).
    stream = np.random.default_rng(100 + rank).integers(1, spec.vocab_size, size=W_ + K_ + 1).tolist()

    def make_engine(graphs=True):
        rt = OffloadRuntime(dw, slots, lookahead=2)
        persistent = None if os.environ.get("MOBILE_PERSISTENT", "") == "" else os.environ["MOBILE_PERSISTENT"] != "0"
        eng = StepEngine(dm, 1, max_len, runtime=rt, graphs=graphs, persistent=persistent).build(gamma=policy.gamma)
        return rt, eng

    def timed_decode(full: bool, natural: bool = False):
        """natural: the confidence rule decides the fallbacks (policy.py:69-79)
        instead of the injected flags"""
        rt, eng = make_engine()
        eng.prefill(prompt)
        for i in range(W_):
            eng.step(None if natural else flags[i], full=full, next_token=stream[i])
        torch.cuda.synchronize()
        barrier(ws)
        launches0 = K.LAUNCHES[0]
        bytes0, xfer0 = rt.counters()
        stats0 = rt.cache.stats
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            ev0.record(eng.stream)
            w0 = time.perf_counter()
            fb = 0
            for i in range(W_, W_ + K_):
                _, f = eng.step(None if natural else flags[i], full=full, next_token=stream[i])
                fb += f
            ev1.record(eng.stream)
            torch.cuda.synchronize()
            wall = time.perf_counter() - w0
        dev_s = ev0.elapsed_time(ev1) / 1e3
        bytes1, xfer1 = rt.counters()
        st = rt.cache.stats
        n_graph_kernels = kernels_per_pass(eng, "full" if full else "little")
        out = dict(dev_s=dev_s, wall_s=wall, launches=K.LAUNCHES[0] - launches0, fallbacks=fb,
                   h2d_bytes=bytes1 - bytes0, transfers=xfer1 - xfer0,
                   hits=st.hits - stats0.hits, issued=st.issued - stats0.issued,
                   coalesced=st.coalesced - stats0.coalesced, clocks=clk.summary(), graph_kernels=n_graph_kernels)
        del eng, rt
        torch.cuda.empty_cache()
        return out

    mob = timed_decode(full=False)
    base = timed_decode(full=True)
    nat = timed_decode(full=False, natural=True)

    # isolated PCIe H2D peak (pinned, 1 GiB) for the copy-engine roofline
    hbuf = torch.empty(2**30, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(2**30, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dbuf.copy_(hbuf, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(4):
            dbuf.copy_(hbuf, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    pcie_peak = 4 * 2**30 / (e0.elapsed_time(e1) / 1e3) / 1e9
    del hbuf, dbuf

    # end-to-end: the public decode() call with host inputs (prompt + K teacher-forced ids),
    # including the 512-token prefill, H2D of every input id and D2H of every output id
    rt, eng = make_engine()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    toks, _ = eng.decode(list(prompt), K_, fallback_flags=flags[:K_], inputs=stream[:K_])
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    del eng, rt
    torch.cuda.empty_cache()

    # live roofline of the dominant kernel: the persistent decode-pass kernel on
    # the same shape with every expert HBM-resident (the offload run above is
    # PCIe-bound by design); one graph-replayed pass per kind, CUDA events on
    # the engine stream, inputs (4-5 GB of weights per pass) >> L2
    del dm, dw
    torch.cuda.empty_cache()
    roof = resident_roofline(spec, dev, args.prompt_len, rank)

    dev_s = max_over_ranks(ws, mob["dev_s"], dev)
    base_s = max_over_ranks(ws, base["dev_s"], dev)
    nat_s = max_over_ranks(ws, nat["dev_s"], dev)
    e2e_s = max_over_ranks(ws, e2e_s, dev)
    wall_s = max_over_ranks(ws, mob["wall_s"], dev)
    value = ws * K_ / dev_s
    base_value = ws * K_ / base_s

    P = peaks()
    achieved = roof["little"]["gbs"]
    ep = None
    if not args.no_ep:
        ep = ep_block(args, ws, rank, dev, P)
    per_config = None
    if rank == 0 and not args.no_configs:
        per_config = config_sweep(args, dev, P)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_leg(args, args.cpu_steps or K_, 2)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": ws, "steps": K_,
            "warmup": W_, "ms_per_step": round(dev_s / K_ * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init bf16 weights on the device, random 512-token prompt)",
            "config": bench_config(args, ws, slots, spec.num_layers * spec.num_experts, spec.num_layers),
            "baseline_full_topk": {"value": round(base_value, 3), "unit": "tokens/s",
                                   "ms_per_step": round(base_s / K_ * 1e3, 3), "h2d_bytes": base["h2d_bytes"],
                                   "cache_hits": base["hits"], "transfers": base["transfers"]},
            "speedup_vs_full_topk": round(value / base_value, 4),
            "mobile_natural_r": {"value": round(ws * K_ / nat_s, 3),
                                 "unit": "tokens/s", "fallbacks": nat["fallbacks"],
                                 "r_observed": round(nat["fallbacks"] / K_, 4),
                                 "speedup_vs_full_topk": round(base_s / nat_s, 4),
                                 "note": "same decode with the fallbacks decided by the confidence rule "
                                         "(max p <= gamma = 0.7) on random-init weights instead of the injected "
                                         "paper ratio"},
            "mobile": {"fallbacks": mob["fallbacks"], "h2d_bytes": mob["h2d_bytes"], "transfers": mob["transfers"],
                       "cache_hits": mob["hits"], "cache_coalesced": mob["coalesced"],
                       "wall_ms_per_step": round(mob["wall_s"] / K_ * 1e3, 3)},
            "pcie": {"bound": "pcie_h2d", "achieved_gbs": round(mob["h2d_bytes"] / mob["dev_s"] / 1e9, 2),
                     "peak_gbs": round(pcie_peak, 2), "peak_note": "measured in this run: 1 GiB pinned H2D",
                     "frac": round(mob["h2d_bytes"] / mob["dev_s"] / 1e9 / pcie_peak, 4)},
            "roofline": {"bound": "hbm", "kernel": "decode_pass_kernel (persistent; one resident little pass, "
                                                   "all 24 layers + head in one launch)",
                         "achieved": round(achieved, 1), "peak": P.get("hbm_gbs"), "unit": "GB/s",
                         "frac": round(achieved / P.get("hbm_gbs", 6543.1), 4), "traffic": ncu_traffic(),
                         "launches_timed": roof["little"]["launches"], "bytes_per_launch": roof["little"]["bytes"],
                         "us_per_launch": roof["little"]["us"], "passes": roof,
                         "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(ws * K_ / wall_s, 3), "unit": "tokens/s",
                    "h2d_bytes_per_step": 4,
                    "d2h_bytes_per_step": int(4 + 1 + 4 * (spec.num_experts + 1) * spec.num_layers),
                    "note": "host wall clock of the K timed StepEngine.step() calls (the public per-token API): "
                            "each step's input id H2D from pinned host memory, its token id + fallback flag D2H, "
                            "the C++ cache driver and every expert copy inside"},
            "e2e_incl_prefill": {"value": round(K_ / e2e_s * ws, 3), "unit": "tokens/s",
                                 "note": "wall clock of StepEngine.decode(prompt host list, K) on a cold expert "
                                         "cache, incl. the %d-token prefill" % args.prompt_len},
            "ep": ep,
            "configs": per_config,
            "gpu_launches": mob["launches"] + mob["graph_kernels"] * (K_ + mob["fallbacks"]),
            "clocks": mob["clocks"],
            "init_s": round(t_init, 1),
        }
        print(json.dumps(line), flush=True)


def resident_roofline(spec, dev, ctx, rank):
    """GPU time of one persistent decode pass per kind with resident experts,
    and its algorithmic HBM bytes: per layer qkv + o + router (+ shared-gate
    rows) + k experts + shared experts + the K/V rows read by attention, plus
    the head."""
    import numpy as np
    import torch

    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights
    dw = DeviceWeights.random(spec, dev, seed=rank, experts_on_device=True)
    dm = DeviceModel(dw)
    eng = StepEngine(dm, 1, ctx + 64, persistent=True).build()
    prompt = np.random.default_rng(7).integers(1, spec.vocab_size, size=ctx).tolist()
    eng.prefill(prompt)
    for i in range(4):
        eng.step(False, next_token=i + 11)
    eb, d, L = dw.elem_bytes, spec.hidden_dim, spec.num_layers
    out = {}
    reps = 20
    for kd in ("little", "big", "full"):
        k = eng.k[kd]
        per_layer = (2 * d * d + 2 * d * spec.kv_dim + (spec.num_experts + dw.n_gate_rows) * d) * eb + k * dw.expert_bytes \
            + spec.n_shared * dw.shared_bytes + 2 * (ctx + 4) * spec.kv_dim * 4
        tot = L * per_layer + spec.vocab_size * d * eb
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            e0.record()
            for _ in range(reps):
                eng.graphs[kd].replay()
            e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        out[kd] = {"us": round(us, 1), "bytes": int(tot), "gbs": round(tot / us / 1e3, 1), "launches": reps}
    del eng, dm, dw
    torch.cuda.empty_cache()
    return out


def kernels_per_pass(eng, kind):
    """libmobile kernels inside one captured pass (graph replays are not
    counted by the wrapper counter): the persistent pass is one launch per
    offload segment (L+1) or per resident pass; the per-op engine launches
    qkv, attention, o, router, gate-up, down(+combine) per layer, embed, head."""
    s = eng.spec
    if eng.dp:
        return s.num_layers + 1 if eng.rt is not None else 1
    per_layer = 8 + (2 if s.n_shared else 0)
    return s.num_layers * per_layer + 2


def cpu_leg(args, steps, warmup):
    """The oracle port of the same decode on this host's cores (oracle/ only:
    the product package is never on this path)."""
    from dataclasses import replace

    import numpy as np

    from oracle import cpu_baseline as CB
    from oracle import moe_ref as R
    spec = CB.C3_SPEC if not args.layers else replace(CB.C3_SPEC, num_layers=args.layers)
    W = CB.aliased_weights(spec)
    prompt = np.random.default_rng(1).integers(1, spec.vocab_size, size=1).tolist()
    flags = R.injected_fallback_flags(warmup + steps, args.r)
    from threadpoolctl import threadpool_limits
    n_cores = os.cpu_count() or 1
    with threadpool_limits(limits=n_cores):
        secs, fb = CB.time_decode(W, prompt, flags, warmup, steps, context=args.prompt_len - 1)
    return {"value": round(steps / secs, 4), "unit": "tokens/s", "cores": n_cores, "kind": "port",
            "sample": f"{steps} decode tokens ({fb} fallback, injected r={args.r}) of the same Qwen shape after "
                      f"{warmup} warm-up tokens, context {args.prompt_len} (synthetic KV cache), fp32 NumPy oracle "
                      f"KVDecoder on {n_cores} threads; expert/attention matrices aliased to pools > LLC"}


# ----------------------------------------------------------------------------- expert parallelism
def ep_block(args, ws, rank, dev, P):
    """BASELINE.json C4 (DeepSeek-MoE-16B shape) batched decode, EXPERT-
    PARALLEL over the ws ranks of this launch (ep.EPStepEngine): routed
    experts in contiguous blocks per rank (64 / ws), everything else
    replicated, each rank decoding its own --ep-batch sequences at context
    512; rows exchanged every layer through IPC-mapped peer mailboxes
    (NVLink on a multi-GPU node; at ws = 1 through the rank's own mailbox).
    Pass times are graph replays timed with CUDA events on the engine stream
    (10 each, max over ranks); the exchange legs (dispatch + wait, owner
    experts, return + collect) come from one eager pass with CUDA events
    around each leg.  tokens/s is the whole job: ws x batch per step."""
    import math

    import torch

    from paper_2510_12357_b200.ep import EPStepEngine, ExchangeTimer, partition
    from paper_2510_12357_b200.model import DeviceModel, MoBiLEMoE
    from paper_2510_12357_b200.presets import DEEPSEEK_MOE_16B as spec
    from paper_2510_12357_b200.weights import DeviceWeights

    B, ctx, r = args.ep_batch, 512, 0.11
    group = None
    dw = DeviceWeights.random(spec, dev, seed=0)
    dm = DeviceModel(dw)
    lo, hi = partition(spec.num_experts, ws)[rank]
    local = MoBiLEMoE(dw.shard_experts(lo, hi))
    eng = EPStepEngine(dm, local, B, ctx + 48, group=group).build()
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    eng.sess.kc.normal_(generator=g)
    eng.sess.vc.normal_(generator=g)
    eng.pos.fill_(ctx)
    eng.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device=dev, dtype=torch.int32, generator=g))
    for kd in ("little", "big", "full"):
        eng.graphs[kd].replay()
    torch.cuda.synchronize()

    def time_pass(kd, reps=10):
        barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            e0.record()
            for _ in range(reps):
                eng.graphs[kd].replay()
            e1.record()
        torch.cuda.synchronize()
        return max_over_ranks(ws, e0.elapsed_time(e1) / reps, dev)

    ms = {kd: time_pass(kd) for kd in ("little", "big", "full")}
    # exchange legs: one eager little pass with events around every leg
    eng.use_graphs, eng.ex_timer = False, ExchangeTimer()
    barrier(ws)
    with torch.cuda.stream(eng.stream):
        eng._whole_pass("little")
    legs = eng.ex_timer.summary_ms()
    eng.use_graphs, eng.ex_timer = True, None
    legs = {k: (round(max_over_ranks(ws, v, dev), 3) if k != "exchanges" else v) for k, v in legs.items()}
    p_any = 1.0 - (1.0 - r) ** B
    t_mob = ms["little"] + p_any * ms["big"]  # conservative: the big pass over the whole batch
    eng.close()
    del eng
    # expert-parallel prefill: a 512-token prompt per rank through the session
    # path with every MoE layer's experts exchanged (wall clock, max over ranks)
    pe = EPStepEngine(dm, local, 1, ctx + 8, group=group, graphs=False)
    prompt = torch.randint(1, spec.vocab_size, (ctx + 1,), generator=torch.Generator().manual_seed(5 + rank)).tolist()
    pe.prefill(prompt)  # warm-up (TMA descriptors, the prompt-sized exchange)
    barrier(ws)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    pe.prefill(prompt)
    torch.cuda.synchronize()
    t_pf = max_over_ranks(ws, time.perf_counter() - w0, dev)
    pe.close()
    del pe
    del local, dm, dw
    torch.cuda.empty_cache()
    return {"workload": f"C4 DeepSeek-MoE-16B shape, batched decode, {B} sequences per rank, context {ctx}, "
                        f"expert-parallel over {ws} rank(s) (experts {lo}-{hi - 1} on rank {rank})",
            "parallelism": f"ep{ws}", "batch_per_rank": B, "n_gpus": ws,
            "pass_ms": {k: round(v, 3) for k, v in ms.items()},
            "mobile_tokens_s": round(ws * B / t_mob * 1e3, 1),
            "full_topk_tokens_s": round(ws * B / ms["full"] * 1e3, 1),
            "speedup_vs_full_topk": round(ms["full"] / t_mob, 4), "r": r, "p_any_fallback": round(p_any, 4),
            "exchange_ms_per_little_pass": legs,
            "prefill": {"tokens_per_rank": ctx, "ms": round(t_pf * 1e3, 2), "tokens_s": round(ws * ctx / t_pf, 1),
                        "note": "EPStepEngine.prefill: the prompt through the session path, every MoE layer's "
                                "experts exchanged; wall clock max over ranks"},
            "note": "pass times max over ranks; MoBiLE = little + P(any row falls back) x big (whole-batch replay); "
                    "exchange legs from an eager pass (CUDA events on the engine stream)"}


# ----------------------------------------------------------------------------- other configs
R_PAPER = {"c2": 0.21, "c3": 0.11, "c4": 0.11, "c5": 0.11}  # PAPER.md: OLMoE 0.21, Qwen 0.11
CTX = {"c2": 512, "c3": 512, "c4": 512, "c5": 2048}
BATCHES = {"c2": (1,), "c4": (1, 8, 64, 256), "c5": (1,)}


def config_sweep(args, dev, P):
    """BASELINE.json configs C2 / C4 / C5 at 1 GPU, experts HBM-resident,
    random-init bf16 weights: decode passes (little / replayed big / full
    top-k; graph replays timed with CUDA events on the engine stream, 10
    replays each, inputs >> L2) as MoBiLE tokens/s at the paper's fallback
    ratio vs full-top-k tokens/s, each pass's HBM roofline fraction; C5 also a
    2048-token prefill with its expert GEMMs' tensor roofline fraction; and the
    oracle port's decode on the host cores beside each (CPU legs import
    oracle/ only)."""
    import math
    import numpy as np
    import torch

    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.presets import NAMES, PRESETS
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.weights import DeviceWeights

    hbm, tens = P.get("hbm_gbs", 6543.1), P.get("bf16_tflops", 1403.0)
    out = {}
    for name in [c for c in args.configs.split(",") if c]:
        if name == "c1":
            out[name] = c1_line()
            continue
        spec = PRESETS[name]
        t0 = time.time()
        dw = DeviceWeights.random(spec, dev, seed=0)
        dm = DeviceModel(dw)
        ctx, r = CTX[name], R_PAPER[name]
        res = {"model": NAMES[name], "context": ctx, "r": r, "decode": {}}
        eb, d, L = dw.elem_bytes, spec.hidden_dim, spec.num_layers

        def pass_bytes(e, kd, B):
            """Algorithmic bytes of one pass: every weight the pass needs once,
            routed experts counted as the DISTINCT experts each layer selected
            in this pass (several tokens on one expert read it once)."""
            idx = e.idx[kd][:, :B, :e.k[kd]].reshape(L, -1)
            distinct = int(sum(torch.unique(idx[l]).numel() for l in range(L)))
            per_layer = (2 * d * d + 2 * d * spec.kv_dim + (spec.num_experts + dw.n_gate_rows) * d) * eb \
                + spec.n_shared * dw.shared_bytes + B * 2 * ctx * spec.kv_dim * 4
            return L * per_layer + distinct * dw.expert_bytes + spec.vocab_size * d * eb, distinct

        def engine(B):
            e = StepEngine(dm, B, ctx + 48).build()
            e.sess.kc.normal_()
            e.sess.vc.normal_()
            e.pos.fill_(ctx)
            e.tok.copy_(torch.randint(1, spec.vocab_size, (B,), device=dev, dtype=torch.int32))
            for kd in ("little", "big", "full"):
                e.graphs[kd].replay()
            torch.cuda.synchronize()
            return e

        def time_pass(e, kd, reps=10):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(e.stream):
                e0.record()
                for _ in range(reps):
                    e.graphs[kd].replay()
                e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps / 1e3

        for B in BATCHES[name]:
            eng = engine(B)
            row = {"engine": "gemm" if eng.gemm_path else ("persistent" if eng.dp else "per-op")}
            for kd in ("little", "big", "full"):
                t = time_pass(eng, kd)
                nb, distinct = pass_bytes(eng, kd, B)
                row[kd] = {"ms": round(t * 1e3, 3), "bytes": nb, "distinct_experts": distinct,
                           "gbs": round(nb / t / 1e9, 1), "hbm_frac": round(nb / t / 1e9 / hbm, 4)}
            del eng
            torch.cuda.empty_cache()
            # batched MoBiLE: the big pass replays only the rows that fell back
            p_any = 1.0 - (1.0 - r) ** B
            b_fb = max(1, math.ceil(r * B / p_any - 1e-9))
            if b_fb == B:
                t_big = row["big"]["ms"]
            else:
                e2 = engine(b_fb)
                t_big = round(time_pass(e2, "big") * 1e3, 3)
                del e2
                torch.cuda.empty_cache()
            t_mob = row["little"]["ms"] + p_any * t_big
            row.update({"big_rows": b_fb, "big_rows_ms": t_big, "p_any_fallback": round(p_any, 4),
                        "mobile_tokens_s": round(B * 1e3 / t_mob, 2),
                        "full_topk_tokens_s": round(B * 1e3 / row["full"]["ms"], 2),
                        "speedup_vs_full_topk": round(row["full"]["ms"] / t_mob, 4)})
            res["decode"][f"B{B}"] = row
        if name == "c5":  # 2k-token prefill (per-op engine: attention + tcgen05 grouped-GEMM experts)
            pe = StepEngine(dm, 1, ctx + 8, persistent=False)
            prompt = np.random.default_rng(1).integers(1, spec.vocab_size, size=ctx).tolist()
            pe.prefill(prompt)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            pe.prefill(prompt)
            torch.cuda.synchronize()
            tp = time.perf_counter() - w0
            I = spec.ffn
            flops = 2.0 * ctx * L * spec.k_big * 3 * d * I
            res["prefill"] = {"tokens": ctx, "ms": round(tp * 1e3, 2), "tokens_s": round(ctx / tp, 1),
                              "expert_gemm_tflop": round(flops / 1e12, 2),
                              "roofline": {"bound": "tensor", "achieved": round(flops / tp / 1e12, 1),
                                           "peak": tens, "unit": "TFLOP/s", "frac": round(flops / tp / 1e12 / tens, 4),
                                           "note": "expert GEMM FLOPs / whole-prefill wall time (attention, "
                                                   "projections and routing included in the time)"}}
            del pe
        res["init_s"] = round(time.time() - t0, 1)
        del dm, dw
        torch.cuda.empty_cache()
        if not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_config_leg(name, r)
        out[name] = res
    return out


def c1_line(n_tokens=24):
    """C1 (the reference's own tiny config, configs[0]): the UNMODIFIED
    reference `moesim.toymoe.generate` (toymoe.py:246-303, staged into
    oracle/_ref by oracle/stage_ref.py) on the host cores next to this
    package's drop-in `generate` on the GPU, identical spec / prompt / policy;
    tokens and accept/fallback decisions must be identical."""
    import sys as _sys

    ref_dir = ROOT / "oracle" / "_ref"
    if not (ref_dir / "moesim" / "toymoe.py").is_file():
        return {"unavailable": "oracle/_ref not staged (python oracle/stage_ref.py in the build container)"}
    _sys.path.insert(0, str(ref_dir))
    try:
        import moesim.config as RC
        import moesim.toymoe as RT
    finally:
        _sys.path.remove(str(ref_dir))
    import paper_2510_12357_b200 as M
    import torch

    kw = dict(num_layers=2, num_experts=16, k_big=4, k_little=2, hidden_dim=256, vocab_size=256, seed=0)
    prompt = [3, 17, 42, 5]
    rm = RT.build_model(RC.ModelSpec(**kw))
    RT.generate(rm, prompt, RC.PolicySpec(), n_tokens)  # warm-up: the same lengths as the timed run
    w0 = time.perf_counter()
    rt, rd = RT.generate(rm, prompt, RC.PolicySpec(), n_tokens)
    t_ref = time.perf_counter() - w0
    om = M.build_model(M.ModelSpec(**kw))
    M.generate(om, prompt, M.PolicySpec(), n_tokens)  # warm-up: every prefix length once (first-shape costs)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ot, od = M.generate(om, prompt, M.PolicySpec(), n_tokens)
    torch.cuda.synchronize()
    t_ours = time.perf_counter() - w0
    same = ot == rt and [d.accepted_by for d in od] == [d.accepted_by for d in rd] and \
        [d.little_selections for d in od] == [d.little_selections for d in rd]
    n = len(rd)
    return {"model": "tiny (SPEC.md): L2 E16 K4 k2 d256 V256, fp64 reference", "tokens": n, "prompt": len(prompt),
            "reference": {"value": round(n / t_ref, 2), "unit": "tokens/s", "impl": "moesim.toymoe.generate "
                          "(unmodified, oracle/_ref)", "cores": os.cpu_count() or 1},
            "ours": {"value": round(n / t_ours, 2), "unit": "tokens/s",
                     "impl": "paper_2510_12357_b200.generate (drop-in API, libmobile kernels)"},
            "fallbacks": sum(d.accepted_by != "Little" for d in rd),
            "identical_tokens_and_decisions": bool(same),
            "note": "wall clock of generate(prompt, max_len) on both sides; the reference recomputes the whole "
                    "prefix per token (no KV cache) and so does the drop-in API"}


def cpu_config_leg(name, r, steps=2, warmup=1):
    """The oracle port's KV decode of config `name` on the host cores (oracle/
    only; matrices aliased to pools larger than the LLC, bounded RAM)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import cpu_baseline as CB
    from oracle import moe_ref as R
    spec = CB.SPECS[name]
    W = CB.aliased_weights(spec, expert_pool=4 if name == "c5" else 64)
    flags = R.injected_fallback_flags(warmup + steps, r)
    n_cores = os.cpu_count() or 1
    with threadpool_limits(limits=n_cores):
        secs, fb = CB.time_decode(W, [1], flags, warmup, steps, context=CTX[name])
    return {"value": round(steps / secs, 4), "unit": "tokens/s", "cores": n_cores, "kind": "port",
            "sample": f"{steps} decode tokens ({fb} fallback, injected r={r}) after {warmup} warm-up, context "
                      f"{CTX[name]} (synthetic KV cache), fp32 NumPy oracle KVDecoder"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, ws, rank):
    """The reference's CPU path of the same decode: the oracle port (the
    reference package cannot build d=2048 models, toymoe.py:100-107), every
    host core, the same metric / unit / config.  Imports oracle/ only."""
    if rank != 0:
        return
    from oracle import cpu_baseline as CB
    slots = CB.c3_slots(int(args.cap_gib * 2**30), int(args.reserved_gib * 2**30))
    spec = CB.C3_SPEC
    cpu = cpu_leg(args, args.steps, args.warmup)
    v = cpu["value"]
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 / v, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "impl": "reference",
            "data": "synthetic (random-init fp32 weights, synthetic 512-position KV context)",
            "config": bench_config(args, ws, slots, spec.num_layers * spec.num_experts, spec.num_layers),
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, ws, rank)
        return
    ws, rank, local = dist_init(args)
    if os.environ.get("MOBILE_BENCH_SHARE_GPU") == "1":
        local = 0
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
