"""Scorer throughput vs available parallelism: the C2 feeder with its 24
scenarios replicated k times (L = 24k), first 10% of the reduction, host loop
with per-launch CUDA-event timing of the scorer."""
import sys, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2510_19608_b200 as kr
from golden_io import path

src = path("c2", "scen.csv").read_text().splitlines()
hdr, body = src[0], src[1:]
for k in [int(x) for x in sys.argv[1:]] or [1, 2, 4]:
    lines = [hdr]
    for rep in range(k):
        for ln in body:
            f = ln.split(",")
            scale = 1.0 + 0.01 * rep
            lines.append(",".join([f"{f[0]}_{rep}", f[1], f[2], repr(float(f[3]) * scale), repr(float(f[4]) * scale)]))
    d = Path(tempfile.mkdtemp())
    (d / "scen.csv").write_text("\n".join(lines) + "\n")
    ctx = kr.Context(kr.HostProblem(str(path("c2", "net.json")), str(d / "scen.csv")), device=0)
    cfg = kr.ReductionConfig(e_bar=3e-3, target_reduction=0.1)
    ctx.run_reduction(cfg)
    ctx.set_profile(True)
    res = ctx.run_reduction(cfg)
    st = ctx.kernel_stats(0)
    pr = sum(t.candidate_count * (t.supernode_count + 1) for t in res.trace) * 24 * k
    us = 1e3 * st["ms"] / st["launches"]
    print(f"L={24*k:4d}: score avg {us:7.1f} us/launch, {pr / (st['ms'] * 1e-3) / 1e9:6.2f} G pair-rows/s")
