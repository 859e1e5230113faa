"""Spec/config mirror and host-side plan bookkeeping (CPU)."""
import numpy as np
import pytest

from paper_2510_12357_b200 import (ConfigError, HardwareSpec, ModelSpec, PolicySpec, data_path, hbm_expert_slots,
                                   injected_fallback_flags, load_config_file, parse_bytes)
from paper_2510_12357_b200.policy import PlanEntry, plan_from_targets, on_demand_selection
from paper_2510_12357_b200.spec import ExpertId


def test_parse_bytes():
    assert parse_bytes("64MiB") == 64 * 2**20
    assert parse_bytes("16GiB/s") == 16 * 2**30
    assert parse_bytes("2KB") == 2000
    assert parse_bytes(5) == 5
    for bad in ("x", "5QB", True, -1):
        with pytest.raises(ConfigError):
            parse_bytes(bad)


def test_packaged_slots(golden):
    meta, _ = golden
    m = load_config_file(data_path("olmoe_desk.json"))["model"]
    hw = load_config_file(data_path("rtx4080.json"))["hardware"]
    assert hbm_expert_slots(m, hw) == meta["slots_packaged"] == 158
    pol = load_config_file(data_path("policy_default.json"))["policy"]
    assert pol.gamma == 0.7 and pol.reuse_little_gates is False


def test_validation_messages():
    with pytest.raises(ConfigError, match="exceeds num_experts"):
        ModelSpec(num_layers=1, num_experts=4, k_big=5).validate()
    with pytest.raises(ConfigError, match="k_little"):
        ModelSpec(num_layers=1, num_experts=4, k_big=2, k_little=3).validate()
    with pytest.raises(ConfigError, match="gamma"):
        PolicySpec(gamma=1.5).validate()
    with pytest.raises(ConfigError, match="lookahead"):
        HardwareSpec(lookahead_depth=0).validate()
    assert ModelSpec(num_layers=1, num_experts=8, k_big=4).k_little == 2
    assert ModelSpec(num_layers=1, num_experts=8, k_big=1).k_little == 1


def test_unknown_fields_rejected(tmp_path):
    p = tmp_path / "c.json"
    p.write_text('{"model": {"num_layers": 1, "num_experts": 2, "k_big": 1, "bogus": 3}}')
    with pytest.raises(ConfigError, match="unknown fields"):
        load_config_file(p)


def test_injected_flags(golden):
    meta, _ = golden
    for c in meta["injected"]:
        assert injected_fallback_flags(c["n"], c["r"]) == c["flags"]
    with pytest.raises(ValueError):
        injected_fallback_flags(10, 1.5)


def test_plan_windows_and_order(golden):
    """Host bookkeeping of build_mobile_plan given the reference's own targets."""
    meta, _ = golden
    for c in meta["plans"]:
        targets = [[e for (_, e) in row] for row in c["targets"]]
        plan = plan_from_targets(targets, c["lookahead"])
        assert [[e.earliest_issue_layer, e.expert.layer, e.expert.expert, e.after_routing] for e in plan.entries] == c["entries"]


def test_on_demand_plan():
    sel = [[ExpertId(0, 1)], [ExpertId(1, 0), ExpertId(1, 3)]]
    plan = on_demand_selection(sel)
    assert all(e.after_routing and e.earliest_issue_layer == e.expert.layer for e in plan.entries)
    sel[0].append(ExpertId(0, 2))
    assert plan.targets[0] == [ExpertId(0, 1)]
    with pytest.raises(ValueError, match="layer 1"):
        on_demand_selection([[ExpertId(0, 0)], []])


def test_bench_reference_arm_restates_the_bench_workload():
    """bench.py --impl reference imports only oracle/: its restated C3 shape
    and slot count must be the product's (same_config on both arms)."""
    from oracle import cpu_baseline as CB
    from paper_2510_12357_b200 import HardwareSpec, hbm_expert_slots
    from paper_2510_12357_b200.presets import QWEN15_MOE, with_byte_sizes
    assert CB.C3_SPEC == CB.oracle_spec_from(QWEN15_MOE)
    for cap, res in ((16, 6), (8, 2)):
        hw = HardwareSpec(hbm_capacity=cap * 2**30, reserved=res * 2**30)
        assert CB.c3_slots(cap * 2**30, res * 2**30) == hbm_expert_slots(with_byte_sizes(QWEN15_MOE), hw)


def test_oracle_bench_specs_match_presets():
    """bench.py's CPU legs build the config shapes on the oracle side
    (oracle/cpu_baseline.SPECS, no product import); they must equal presets.py."""
    from oracle import cpu_baseline as CB
    from paper_2510_12357_b200.presets import PRESETS
    for name, spec in CB.SPECS.items():
        assert CB.oracle_spec_from(PRESETS[name]) == spec, name
