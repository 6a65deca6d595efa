import sys, time
sys.path[:0] = ['/root/repo', '/root/repo/tests']
import paper_2510_19608_b200 as kr
from golden_io import path
for case, tgt in (("c3", 0.1), ("c4", 0.1)):
    ctx = kr.Context(kr.HostProblem(str(path(case, "net.json")), str(path(case, "scen.csv"))), device=0)
    cfg = kr.ReductionConfig(e_bar=3e-3, target_reduction=tgt)
    r = ctx.run_reduction(cfg)
    print(case, "plain run", len(r.trace), "iters", round(r.device_ms, 1), "ms", round(r.device_ms / len(r.trace) * 1e3, 1), "us/iter")
    ctx.set_profile(True)
    r = ctx.run_reduction(cfg)
    sk = ctx.kernel_stats(0); sv = ctx.kernel_stats(1)
    print(case, "profiled", round(r.device_ms, 1), "ms; score", sk["launches"], round(1e3 * sk["ms"] / sk["launches"], 1), "us/launch; base", sv["launches"], round(1e3 * sv["ms"] / max(1, sv["launches"]), 1), "us/launch")
