"""C3 offloaded-decode operating points beside the headline (SURVEY.md §8d:
the second cache budget and the injected fallback ratios): one bench.py run
per point, summarised into one JSON object.
    python scripts/c3_points.py > profiles/r2_c3_points.json"""
import json
import subprocess
import sys

POINTS = ["--cap-gib 8 --reserved-gib 2", "--r 0", "--r 0.21", "--r 1.0"]
BASE = "--no-cpu-baseline --no-configs --no-ep --steps 48 --warmup 12"
out = {"source": f"python bench.py {BASE} <args> (C3 offloaded decode, 1 B200); the headline point "
                 "(477 slots, r=0.11) is profiles/r2_bench_line.json", "points": []}
for args in POINTS:
    r = subprocess.run([sys.executable, "bench.py", *BASE.split(), *args.split()], capture_output=True, text=True)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode or not lines:
        out["points"].append({"args": args, "error": r.stderr[-400:]})
        continue
    d = json.loads(lines[-1])
    out["points"].append({"args": args, "slots": d["config"]["hbm_expert_slots"], "r": d["config"]["r_injected"],
                          "mobile_tok_s": d["value"], "full_topk_tok_s": d["baseline_full_topk"]["value"],
                          "speedup": d["speedup_vs_full_topk"], "pcie_frac": d["pcie"]["frac"],
                          "fallbacks": d["mobile"]["fallbacks"], "clocks": d.get("clocks")})
    print(json.dumps(out["points"][-1]), file=sys.stderr, flush=True)
print(json.dumps(out))
