"""A/B of scorer settings on a large feeder (env settings in subprocesses):
python tools/large_ab.py c4 24 0.1 "KRONRED_NO_S1=1" "" "KRONRED_S1_GK=16,16,8" ...
Prints one JSON line per setting: device time of one reduction to the target."""
import json, os, subprocess, sys, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
case, L, target = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
settings = sys.argv[4:] or [""]
n = {"c3": 5991, "c4": 8381}[case]
d = Path(tempfile.mkdtemp())
scen = d / "scen.csv"
if L == 2:
    sys.path[:0] = [str(ROOT / "tests")]
    from golden_io import path
    scen = path(case, "scen.csv")
else:
    subprocess.run([str(ROOT / "oracle" / "_ref" / "kronred_ref"), "gen", "--n", str(n), "--seed", str(n), "--L", str(L),
                    "--branching", "0.3", "--net", str(d / "net.json"), "--scen", str(scen)], check=True, capture_output=True)
code = f"""
import sys, json; sys.path[:0] = [{str(ROOT)!r}, {str(ROOT / 'tests')!r}]
import paper_2510_19608_b200 as kr
from golden_io import path
ctx = kr.Context(kr.HostProblem(str(path({case!r}, 'net.json')), {str(scen)!r}), device=0)
r = ctx.run_reduction(kr.ReductionConfig(e_bar=3e-3, target_reduction={target}))
print(json.dumps({{'iterations': len(r.trace), 'device_ms': r.device_ms, 'last_s': r.trace[-1].s, 'last_r': r.trace[-1].r}}))
"""
for s in settings:
    env = dict(os.environ)
    for kv in s.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(json.dumps({"case": case, "L": L, "target": target, "setting": s, **json.loads(out.stdout.strip().splitlines()[-1])}) if out.returncode == 0 else json.dumps({"setting": s, "error": out.stderr[-500:]}), flush=True)
