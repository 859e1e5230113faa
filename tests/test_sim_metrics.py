"""Traces, timing model and metrics vs golden vectors from the
unmodified reference (tests/golden/make_golden_sim.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLD / "sim_golden.json").read_text())


def _setup():
    from paper_2510_12357_b200.spec import HardwareSpec, ModelSpec, PolicySpec
    model = ModelSpec(num_layers=4, num_experts=16, k_big=4, k_little=2, expert_bytes=10 * 1024**2,
                      dense_bytes_per_layer=1024**2)
    hw = HardwareSpec(hbm_capacity=12 * 10 * 1024**2 + 4 * 1024**2 + 1024**2, reserved=1024**2,
                      pcie_bandwidth=16 * 1024**3, pcie_fixed_latency=1e-4, gpu_expert_compute=3e-4,
                      gpu_attn_compute=2.7e-3, lookahead_depth=2)
    return model, hw, PolicySpec(gamma=0.7)


def test_synthetic_trace_bit_identical():
    from paper_2510_12357_b200.trace import SyntheticTraceConfig, gen_synthetic, load_trace
    ref = load_trace(GOLD / "trace_small.jsonl")
    ours = gen_synthetic(SyntheticTraceConfig(seed=3, num_layers=4, num_experts=16, k_big=4, popularity_skew=0.8,
                                              reuse_prob=0.3), 40)
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert a.token_index == b.token_index and a.confidence == b.confidence
        assert np.array_equal(a.layers, b.layers)


def test_trace_roundtrip_and_errors(tmp_path):
    from paper_2510_12357_b200.spec import ConfigError
    from paper_2510_12357_b200.trace import load_trace, save_trace
    recs = load_trace(GOLD / "trace_small.jsonl")
    for name in ("t.jsonl", "t.jsonl.gz"):
        save_trace(tmp_path / name, recs)
        back = load_trace(tmp_path / name)
        assert all(np.array_equal(a.layers, b.layers) and a.confidence == b.confidence for a, b in zip(recs, back))
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"t": 0, "confidence": 0.5}\n')
    with pytest.raises(ConfigError, match="missing key 'layers'"):
        load_trace(bad)
    bad.write_text('{"t": 0, "confidence": 1.5, "layers": [[1.0, 2.0]]}\n')
    with pytest.raises(ConfigError, match="outside"):
        load_trace(bad)


def test_calibration_trace_matches_reference():
    from paper_2510_12357_b200.trace import calibration_trace
    cal = calibration_trace()
    g = G["calibration"]
    assert len(cal) == g["n"]
    assert cal[0].layers[0, :8].tolist() == g["first"] and cal[0].confidence == g["conf0"]
    assert float(sum(r.layers.sum() for r in cal)) == g["sum"]
    assert float(sum(r.confidence for r in cal)) == g["conf_sum"]


def test_analytic_and_csv(tmp_path):
    from paper_2510_12357_b200.metrics import RunMetrics, analytic_speedup, write_metrics_csv
    assert [analytic_speedup(2.0, 1.0, 2.5, 0.2), analytic_speedup(3.0, 1.5, 0.0, 0.0)] == G["analytic"]
    with pytest.raises(ValueError, match="positive"):
        analytic_speedup(0.0, 1.0, 1.0, 0.1)
    rows = [RunMetrics(*[int(v) if i == 1 else v for i, v in enumerate(r)]) for r in G["gamma_sweep"][1:3]]
    # the golden CSV was written for gammas 0.5, 0.9: rebuild its rows from the text and re-emit
    lines = G["csv"].strip().splitlines()
    parsed = [RunMetrics(*[int(x) if i == 1 else float(x) for i, x in enumerate(l.split(","))]) for l in lines[1:]]
    write_metrics_csv(tmp_path / "m.csv", parsed)
    assert (tmp_path / "m.csv").read_text() == G["csv"]
    assert rows


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["conf", "inject"])
def test_run_pair_matches_reference(cuda_ok, name):
    from paper_2510_12357_b200.metrics import run_pair
    from paper_2510_12357_b200.policy import injected_fallback_flags
    from paper_2510_12357_b200.spec import derive_costs, hbm_expert_slots
    from paper_2510_12357_b200.trace import load_trace
    model, hw, pol = _setup()
    recs = load_trace(GOLD / "trace_small.jsonl")
    assert hbm_expert_slots(model, hw) == G["slots"]
    c = derive_costs(model, hw)
    assert [c.t_xfer, c.t_exp, c.t_attn] == G["costs"]
    flags = None if name == "conf" else injected_fallback_flags(len(recs), 0.3)
    base, prim, row = run_pair(recs, model, hw, pol, fallback_flags=flags)
    g = G[f"pair_{name}"]
    assert [t.total for t in base] == g["base_totals"]
    assert [t.fallback for t in prim] == g["prim_fallback"]
    got = [[[p.label, p.total, p.compute, p.transfer_stall, p.overlapped_transfer, p.fresh_transfers, p.hits,
             p.misses] for p in t.passes] for t in prim]
    assert got == g["prim"]
    assert [float(v) for v in row.row()] == g["row"]


@pytest.mark.gpu
def test_sweeps_events_full_mobile_match_reference(cuda_ok):
    from paper_2510_12357_b200.metrics import gamma_sweep, little_size_sweep, run_pair
    from paper_2510_12357_b200.sim import PLAN_MOBILE, simulate_full_stream
    from paper_2510_12357_b200.spec import derive_costs
    from paper_2510_12357_b200.trace import load_trace
    model, hw, pol = _setup()
    recs = load_trace(GOLD / "trace_small.jsonl")
    assert [[float(v) for v in r.row()] for r in gamma_sweep(recs, model, hw, pol, [0.0, 0.5, 0.7, 1.0])] == G["gamma_sweep"]
    assert [[float(v) for v in r.row()] for r in little_size_sweep(recs, model, hw, pol, [1, 2, 3, 4])] == G["little_sweep"]
    full, _ = simulate_full_stream(recs, derive_costs(model, hw), G["slots"], 4, plan_mode=PLAN_MOBILE, lookahead=2)
    assert [t.total for t in full] == G["full_mobile_totals"]
    ev: list = []
    run_pair(recs[:3], model, hw, pol, event_log=ev)
    assert [[t, k, e, l] for t, k, e, l in ev] == G["events"]


@pytest.mark.gpu
def test_measured_metrics_and_trace_export(cuda_ok, tmp_path):
    """Measured B200 passes through the reference's aggregate / CSV contract,
    and the run's exported trace replayed by the timing model."""
    from paper_2510_12357_b200.metrics import aggregate, calibrated_hardware, measure_stream, run_pair, write_metrics_csv
    from paper_2510_12357_b200.offload import OffloadRuntime
    from paper_2510_12357_b200.policy import injected_fallback_flags
    from paper_2510_12357_b200.runtime import StepEngine
    from paper_2510_12357_b200.spec import ModelSpec, PolicySpec
    from paper_2510_12357_b200.trace import load_trace, record_from_engine, save_trace
    from tests.helpers import QWEN_MINI, matched
    from tests.test_runtime_gpu import _offload_dm
    o, ms, dm0 = matched(QWEN_MINI, "bfloat16")
    n = 10
    flags = injected_fallback_flags(n, 0.3)
    runs = {}
    for full in (True, False):
        dm = _offload_dm(dm0, ms)
        rt = OffloadRuntime(dm.dw, slots=8, lookahead=2)
        eng = StepEngine(dm, 1, 64, runtime=rt).build(gamma=0.7)
        runs[full] = measure_stream(eng, [3, 17, 42, 7], n, fallback_flags=None if full else flags, full=full)
    base, prim = runs[True][0], runs[False][0]
    assert all(len(t.passes) == (2 if t.fallback else 1) for t in prim)
    row = aggregate(base, prim, 0.7, ms.k_little)
    assert row.fallback_ratio == sum(flags) / n and 0.0 <= row.cache_hit_rate <= 1.0 and row.speedup_measured > 0
    write_metrics_csv(tmp_path / "measured.csv", [row])
    assert (tmp_path / "measured.csv").read_text().splitlines()[0].startswith("gamma,k_little,fallback_ratio,T,")
    recs = record_from_engine(runs[False][1], runs[False][2])
    save_trace(tmp_path / "b200.jsonl.gz", recs)
    back = load_trace(tmp_path / "b200.jsonl.gz")
    spec = ModelSpec(num_layers=ms.num_layers, num_experts=ms.num_experts, k_big=ms.k_big, k_little=ms.k_little,
                     expert_bytes=dm0.dw.expert_bytes, dense_bytes_per_layer=1)
    hw = calibrated_hardware(spec, 50.0, 2e-6, 4e-6)
    hw = type(hw)(**{**hw.__dict__, "hbm_capacity": 8 * dm0.dw.expert_bytes + spec.num_layers + hw.reserved})
    _, _, pred = run_pair(back, spec, hw, PolicySpec(gamma=0.7), fallback_flags=flags)
    assert pred.fallback_ratio == row.fallback_ratio and pred.speedup_analytic > 0


def test_cli_gen_trace_matches_reference_calibration(tmp_path):
    from paper_2510_12357_b200.cli import main
    from paper_2510_12357_b200.trace import load_trace
    assert main(["gen-trace", "--n", "3", "--out", str(tmp_path / "t.jsonl")]) == 0
    recs = load_trace(tmp_path / "t.jsonl")
    assert len(recs) == 3 and recs[0].layers[0, :8].tolist() == G["calibration"]["first"]


@pytest.mark.gpu
def test_cli_run_trace_and_sweep(cuda_ok, tmp_path):
    from paper_2510_12357_b200.cli import main
    tr = str(GOLD / "trace_small.jsonl")
    model = tmp_path / "model.json"
    model.write_text(json.dumps({"model": {"num_layers": 4, "num_experts": 16, "k_big": 4, "k_little": 2,
                                           "expert_bytes": 10 * 1024**2, "dense_bytes_per_layer": 1024**2}}))
    hw = tmp_path / "hw.json"
    hw.write_text(json.dumps({"hardware": {"hbm_capacity": 12 * 10 * 1024**2 + 4 * 1024**2 + 1024**2,
                                           "reserved": 1024**2, "pcie_bandwidth": 16 * 1024**3,
                                           "pcie_fixed_latency": 1e-4, "gpu_expert_compute": 3e-4,
                                           "gpu_attn_compute": 2.7e-3, "lookahead_depth": 2}}))
    out = tmp_path / "o"
    assert main(["run-trace", "--trace", tr, "--model", str(model), "--hw", str(hw), "--out", str(out),
                 "--event-log"]) == 0
    lines = (out / "metrics.csv").read_text().splitlines()
    assert lines[0] == "gamma,k_little,fallback_ratio,T,T_l,T_b,speedup_measured,speedup_analytic,stall_share,cache_hit_rate"
    assert [float(x) for x in lines[1].split(",")] == G["pair_conf"]["row"]
    assert (out / "events.log").exists() and (out / "manifest.json").exists()
    assert main(["sweep", "--kind", "gamma", "--grid", "0.0,0.5,0.7,1.0", "--trace", tr, "--model", str(model),
                 "--hw", str(hw), "--out", str(out)]) == 0
    rows = (out / "sweep.csv").read_text().splitlines()[1:]
    assert [[float(x) for x in r.split(",")] for r in rows] == G["gamma_sweep"]
