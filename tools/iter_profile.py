"""Per-iteration device timeline of one device-loop reduction.

Runs a golden case with KRONRED_LOOP_TRACE (globaltimer stamps inside the
loop graph) and prints, per iteration bucket, the scorer time against the
candidate count, active rows and pair-rows, so the scorer's throughput- and
latency-bound regimes can be told apart.

  python tools/iter_profile.py [case] [e_bar] [target] [--out file.tsv]
"""
import argparse
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
ap.add_argument("target", nargs="?", type=float, default=None)
ap.add_argument("--out", default=None)
ap.add_argument("--bucket", type=int, default=50)
args = ap.parse_args()

dump = os.path.join(tempfile.mkdtemp(), "stamps.bin")
os.environ["KRONRED_LOOP_TRACE"] = "1"
os.environ["KRONRED_LOOP_TRACE_DUMP"] = dump

import paper_2510_19608_b200 as kr  # noqa: E402
from golden_io import path  # noqa: E402

ctx = kr.Context(kr.HostProblem(str(path(args.case, "net.json")), str(path(args.case, "scen.csv"))), device=0)
cfg = kr.ReductionConfig(e_bar=args.e_bar, target_reduction=args.target)
ctx.run_reduction(cfg)  # graph instantiation
res = ctx.run_reduction(cfg)
T = np.fromfile(dump, dtype=np.uint64).reshape(-1, 16).astype(np.int64)
it = len(res.trace)
L = len(res.trace[0].max_err) if it else 0
rows = []
for i in range(1, it - 1):
    c, nx = T[i], T[i + 1]
    score = (c[0] - c[6]) / 1e3
    pick = (c[1] - c[0]) / 1e3
    after = (nx[6] - c[1]) / 1e3  # pick end -> next score start (enum || refresh)
    C = res.trace[i].candidate_count
    ns = res.trace[i].supernode_count + 1  # before the commit
    # next iteration's enum / refresh phases, relative to this pick's end
    en = (nx[3] - c[1]) / 1e3
    rs, rst, rwk, rbw, re0, rel = [(nx[k] - c[1]) / 1e3 for k in (4, 8, 9, 11, 5, 10)]
    rows.append((i, C, ns, score, pick, after, en, rs, rst, rwk, re0, rel, rbw))
a = np.array(rows)
print(f"{args.case}: {it} iterations, L={L}, total device {res.device_ms:.1f} ms")
print(" iters      C_avg   ns_avg  score_us  pick_us  enum|refresh_us  Mpair-rows/us")
for b0 in range(0, len(a), args.bucket):
    s = a[b0:b0 + args.bucket]
    pr = (s[:, 1] * s[:, 2] * L).mean()
    print(f"{int(s[0,0]):4d}-{int(s[-1,0]):4d} {s[:,1].mean():8.0f} {s[:,2].mean():8.0f} {s[:,3].mean():9.1f} "
          f"{s[:,4].mean():8.1f} {s[:,5].mean():14.1f} {pr / s[:,3].mean() / 1e6:12.3f}")
print(f"sum: score {a[:,3].sum()/1e3:.1f} ms, pick {a[:,4].sum()/1e3:.1f} ms, enum|refresh {a[:,5].sum()/1e3:.1f} ms")
m = a[:, 6:].mean(axis=0)
print(f"after pick (us, mean): enum end {m[0]:.1f} | refresh start {m[1]:.1f}, staged {m[2]:.1f}, "
      f"walk done {m[3]:.1f}, backward done {m[6]:.1f}, CTA0 end {m[4]:.1f}, last CTA end {m[5]:.1f} | next score {a[:,5].mean():.1f}")
se = np.array([(T[i][0] - T[i][15]) / 1e3 for i in range(1, it - 1) if T[i][15] > 0])
if len(se):
    print(f"score1 last CTA end -> pick start: mean {se.mean():.2f} us, median {np.median(se):.2f} us")
s3 = np.array([(T[i][0] - T[i][14]) / 1e3 for i in range(1, it - 1) if T[i][14] > 0])
if len(s3):
    print(f"score3 last CTA end -> pick start: mean {s3.mean():.2f} us, median {np.median(s3):.2f} us, "
          f"score3 ends after score1 in {np.mean([T[i][14] > T[i][15] for i in range(1, it - 1)]) * 100:.0f} % of iterations")
pk = T[2:it, 12]
if pk.any():
    f = lambda sh: np.median((pk >> sh) & 0xFFFF)
    print("pick phases (SM cycles, median): argmin %d, trace %d, commit %d, active-list %d" % (f(0), f(16), f(32), f(48)))
if args.out:
    np.savetxt(args.out, a, fmt="%.3f", delimiter="\t",
               header="iter\tC\tns\tscore_us\tpick_us\tafter_us\tenum_end\tref_start\tref_staged\tref_walk\tref_end0\tref_end\tref_bwd")
