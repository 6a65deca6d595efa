"""Run one reduction of a golden case (default: the 1000-node benchmark feeder)
for profilers: `ncu ... python tools/profile_run.py [case] [e_bar] [target]`."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr  # noqa: E402
from golden_io import path  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2"
e_bar = float(sys.argv[2]) if len(sys.argv) > 2 else 3e-3
target = float(sys.argv[3]) if len(sys.argv) > 3 else None
ctx = kr.Context(kr.HostProblem(str(path(case, "net.json")), str(path(case, "scen.csv"))), device=0)
res = ctx.run_reduction(kr.ReductionConfig(e_bar=e_bar, target_reduction=target))
print(f"{case}: {len(res.trace)} iterations, {res.total_candidates} candidates, {res.device_ms:.1f} ms")
