"""Base refresh timing (full sweep, and the incremental walk with the first
candidate's (s, r)): average per launch over 200 launches and the phase
clocks (kept init, forward, backward) of one launch."""
import ctypes as C, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr
from golden_io import path
case = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = kr.Context(kr.HostProblem(str(path(case, "net.json")), str(path(case, "scen.csv"))), device=0)
ctx.loop_begin(kr.ReductionConfig(e_bar=3e-3))
ctx.loop_candidates()
L = kr.lib()
L.krg_debug_base_refresh.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.c_longlong * 4]
for name, reps in (("full", 200), ("incremental", -200)):
    ms = C.c_double(); clk = (C.c_longlong * 4)()
    rc = L.krg_debug_base_refresh(ctx._h, reps, C.byref(ms), clk)
    print(case, name, "rc", rc, "base refresh %.1f us" % (ms.value * 1e3), "phases (cycles): kept", clk[1] - clk[0],
          "forward", clk[2] - clk[1], "backward", clk[3] - clk[2])
