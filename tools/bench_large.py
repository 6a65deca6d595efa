"""Large-feeder runs (BASELINE configs[2..4] shapes): full GPU reductions on
the committed 5,991-node and 8,381-node feeders (2 scenarios) to the paper's
targets, device time per run and candidates/s. With oracle/_ref present it
also generates the 24- and 96-scenario libraries of the same feeders with the
reference generator (current-mode CSV, bit-identical reload)."""
import json, subprocess, sys, tempfile, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr
from golden_io import path

REF = ROOT / "oracle" / "_ref" / "kronred_ref"
cases = [("c3", 5991, 0.9), ("c4", 8381, 0.8)]
out = []
for case, n, target in cases:
    libs = [("L2", str(path(case, "scen.csv")))]
    if REF.exists() and "--quick" not in sys.argv:
        d = Path(tempfile.mkdtemp())
        for L in (24, 96):
            subprocess.run([str(REF), "gen", "--n", str(n), "--seed", str(n), "--L", str(L), "--branching", "0.3",
                            "--net", str(d / "net.json"), "--scen", str(d / f"scen{L}.csv")], check=True,
                           capture_output=True)
            libs.append((f"L{L}", str(d / f"scen{L}.csv")))
    for name, scen in libs:
        t0 = time.perf_counter()
        ctx = kr.Context(kr.HostProblem(str(path(case, "net.json")), scen), device=0)
        t1 = time.perf_counter()
        cfg = kr.ReductionConfig(e_bar=3e-3, target_reduction=target)
        res = ctx.run_reduction(cfg)
        t2 = time.perf_counter()
        rec = {"case": case, "nodes": n, "scenarios": name, "target": target, "iterations": len(res.trace),
               "candidates": res.total_candidates, "device_ms": res.device_ms,
               "cand_per_s": res.total_candidates / (res.device_ms / 1e3), "create_s": t1 - t0, "run_wall_s": t2 - t1,
               "final_max_err": [float(e) for e in res.model.final_max_err][:4]}
        print(json.dumps(rec), flush=True)
        del ctx
