"""bench.py's JSON-line contract, checked on the CPU through the reference arm
(`--impl reference`: the oracle port of the C3 decode on the host cores).
The GPU arm's keys are checked by the round-end bench itself."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["metric"].startswith("decode tokens/s, MoBiLE vs full-top-k offload baseline")
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    cfg = line["config"]
    assert cfg["context"] == 512 and cfg["hbm_expert_slots"] == 477 and cfg["routed_experts"] == 1440


def test_reference_arm_imports_only_the_oracle():
    """The reference arm must not load the product package (its libmobile.so)."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','1']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "bad=[m for m in sys.modules if m.startswith('paper_2510_12357_b200')]; "
            "print('LOADED', bad); sys.exit(1 if bad else 0)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-1000:] + r.stderr[-2000:]
