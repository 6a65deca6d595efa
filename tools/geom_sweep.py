"""Tuning aid: scorer geometry sweep (Z-column slots per CTA x scenario-slice
width, the KRONRED_S3_G / KRONRED_S3_LS overrides) on a golden case.
`python tools/geom_sweep.py [case] [target] [G:Ls ...] [--L N] [--runs K]`;
prints one JSON line per geometry with the best device time of K (default 3)
reductions. --L N generates an N-scenario library of the 5,991- or 8,381-node
feeder with the reference generator in oracle/_ref (as tools/margin_sweep.py)."""
import json, os, subprocess, sys, tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr  # noqa: E402
from golden_io import path  # noqa: E402

argv = sys.argv[1:]
opt = {}
for k in ("--L", "--runs"):
    if k in argv:
        i = argv.index(k)
        opt[k] = int(argv[i + 1])
        del argv[i:i + 2]
args = [a for a in argv if ":" not in a]
case = args[0] if args else "c2"
target = float(args[1]) if len(args) > 1 else None
geoms = [a for a in argv if ":" in a] or ["16:8", "8:8", "16:4", "32:4", "8:16", "24:4", "12:8"]
scen = str(path(case, "scen.csv"))
if "--L" in opt:
    n = {"c3": 5991, "c4": 8381}[case]
    d = Path(tempfile.mkdtemp())
    scen = str(d / "scen.csv")
    subprocess.run([str(ROOT / "oracle" / "_ref" / "kronred_ref"), "gen", "--n", str(n), "--seed", str(n), "--L",
                    str(opt["--L"]), "--branching", "0.3", "--net", str(d / "net.json"), "--scen", scen],
                   check=True, capture_output=True)
hp = kr.HostProblem(str(path(case, "net.json")), scen)
ref = None
hp_L = opt.get("--L", None)
for g in geoms:
    G, Ls = g.split(":")
    os.environ["KRONRED_S3_G"], os.environ["KRONRED_S3_LS"] = G, Ls
    ctx = kr.Context(hp, device=0)
    cfg = kr.ReductionConfig(e_bar=3e-3, target_reduction=target)
    ms, sig = [], None
    for _ in range(opt.get("--runs", 3)):
        r = ctx.run_reduction(cfg)
        ms.append(r.device_ms)
        sig = [(t.s, t.r, t.smice) for t in r.trace]
    ref = sig if ref is None else ref
    print(json.dumps({"case": case, "L": hp_L, "G": int(G), "Ls": int(Ls), "iterations": len(r.trace),
                      "best_ms": min(ms), "same_decisions": sig == ref}), flush=True)
    del ctx
