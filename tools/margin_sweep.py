"""BASELINE configs[4]: voltage-margin sweep on the 8,381-node feeder with 96
load scenarios, each run to convergence (no reduction target): the
reduction-vs-accuracy curve, with device time and candidates/s per margin.

The 96-scenario library comes from the reference generator in oracle/_ref
(same seed and parameters as the committed 8,381-node feeder). Prints one JSON
line per margin.

  python tools/margin_sweep.py [--margins 0.001,0.002,...] [--case c4]
"""
import argparse
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr  # noqa: E402
from golden_io import path  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--margins", default="0.001,0.002,0.003,0.005,0.01")
ap.add_argument("--case", default="c4")
ap.add_argument("--L", type=int, default=96)
args = ap.parse_args()

REF = ROOT / "oracle" / "_ref" / "kronred_ref"
n = {"c3": 5991, "c4": 8381}[args.case]
d = Path(tempfile.mkdtemp())
scen = d / f"scen{args.L}.csv"
subprocess.run([str(REF), "gen", "--n", str(n), "--seed", str(n), "--L", str(args.L), "--branching", "0.3",
                "--net", str(d / "net.json"), "--scen", str(scen)], check=True, capture_output=True)
hp = kr.HostProblem(str(path(args.case, "net.json")), str(scen))
ctx = kr.Context(hp, device=0)
for e in (float(x) for x in args.margins.split(",")):
    t0 = time.perf_counter()
    res = ctx.run_reduction(kr.ReductionConfig(e_bar=e))
    wall = time.perf_counter() - t0
    ns = n - len(res.trace)
    rec = {"case": args.case, "nodes": n, "scenarios": args.L, "e_bar": e, "iterations": len(res.trace),
           "reduction": 1.0 - ns / n, "kept_nodes": ns, "candidates": res.total_candidates,
           "device_ms": res.device_ms, "cand_per_s": res.total_candidates / (res.device_ms / 1e3),
           "run_wall_s": wall, "final_max_err_max": max(float(v) for v in res.model.final_max_err)}
    print(json.dumps(rec), flush=True)
