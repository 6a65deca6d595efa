"""Tuning aid: scorer row split (lanes per (candidate, scenario) pair,
KRONRED_S3_S = 1 / 2 / 4, or automatic) on a golden case. For each setting:
the best device time of K reductions, and the per-iteration scorer time
(device-loop globaltimer stamps) averaged over iteration buckets, so the
split that wins in each regime (candidate count) can be read off.

  python tools/split_sweep.py [case] [e_bar] [--runs K] [--bucket B] [--S 1,2,4,0]
"""
import argparse
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

ap = argparse.ArgumentParser()
ap.add_argument("case", nargs="?", default="c2")
ap.add_argument("e_bar", nargs="?", type=float, default=3e-3)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--bucket", type=int, default=100)
ap.add_argument("--S", default="1,2,4,0")
ap.add_argument("--fill", default=None)
args = ap.parse_args()
if args.fill:
    os.environ["KRONRED_S3_FILL"] = args.fill

import paper_2510_19608_b200 as kr  # noqa: E402
from golden_io import path  # noqa: E402

hp = kr.HostProblem(str(path(args.case, "net.json")), str(path(args.case, "scen.csv")))
cfg = kr.ReductionConfig(e_bar=args.e_bar)
ref = None
for S in [int(x) for x in args.S.split(",")]:
    os.environ["KRONRED_S3_S"] = str(S)
    os.environ.pop("KRONRED_LOOP_TRACE", None)
    ctx = kr.Context(hp, device=0)
    best = None
    for _ in range(args.runs + 1):
        res = ctx.run_reduction(cfg)
        best = res.device_ms if best is None else min(best, res.device_ms)
    traj = [(t.s, t.r) for t in res.trace]
    ref = ref or traj
    # per-iteration timeline
    dump = os.path.join(tempfile.mkdtemp(), "stamps.bin")
    os.environ["KRONRED_LOOP_TRACE"] = "1"
    os.environ["KRONRED_LOOP_TRACE_DUMP"] = dump
    ctx2 = kr.Context(hp, device=0)
    ctx2.run_reduction(cfg)
    res2 = ctx2.run_reduction(cfg)
    T = np.fromfile(dump, dtype=np.uint64).reshape(-1, 16).astype(np.int64)
    it = len(res2.trace)
    buckets = {}
    for i in range(1, it - 1):
        score = (T[i][0] - T[i][6]) / 1e3
        after = (T[i + 1][6] - T[i][1]) / 1e3
        b = (i // args.bucket) * args.bucket
        buckets.setdefault(b, []).append((score, after, res2.trace[i].candidate_count))
    print(json.dumps({"case": args.case, "S": S, "device_ms": round(best, 2), "same_trajectory": traj == ref,
                      "score_us_by_bucket": {b: round(float(np.mean([x[0] for x in v])), 1) for b, v in buckets.items()},
                      "after_us_by_bucket": {b: round(float(np.mean([x[1] for x in v])), 1) for b, v in buckets.items()},
                      "C_by_bucket": {b: int(np.mean([x[2] for x in v])) for b, v in buckets.items()}}), flush=True)
