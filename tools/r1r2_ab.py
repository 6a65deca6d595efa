"""Round-1 vs current scorer on a large-feeder prefix: runs one reduction of the
8,381-node feeder with a regenerated L-scenario library through the package
found at sys.argv[1] (a checkout root), prints the device time."""
import sys, subprocess, tempfile
from pathlib import Path
root = Path(sys.argv[1]).resolve()
L = int(sys.argv[2]) if len(sys.argv) > 2 else 96
target = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
sys.path[:0] = [str(root), str(root / "tests")]
import paper_2510_19608_b200 as kr
from golden_io import path
scen = Path(tempfile.gettempdir()) / f"c4_L{L}.csv"
if not scen.exists():
    ref = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "kronred_ref"
    d = Path(tempfile.mkdtemp())
    subprocess.run([str(ref), "gen", "--n", "8381", "--seed", "8381", "--L", str(L), "--branching", "0.3",
                    "--net", str(d / "net.json"), "--scen", str(scen)], check=True, capture_output=True)
ctx = kr.Context(kr.HostProblem(str(path("c4", "net.json")), str(scen)), device=0)
cfg = kr.ReductionConfig(e_bar=3e-3, target_reduction=target)
ctx.run_reduction(cfg)
if "--profile" in sys.argv:  # host-driven loop with per-kernel CUDA events
    ctx.set_profile(True)
r = ctx.run_reduction(cfg)
print(root.name, f"L={L}", len(r.trace), "iterations", f"{r.device_ms:.1f} ms")
if "--profile" in sys.argv:
    for k, name in ((0, "scorer"), (1, "base refresh"), (2, "score3 multi")):
        try:
            st = ctx.kernel_stats(k)
            print(f"   {name}: {st['launches']} launches, {st['ms']:.1f} ms")
        except Exception as e:
            print("  ", name, "n/a")
