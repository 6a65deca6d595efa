"""Breakdown of the e2e call (bench.py e2e leg): reload from host, the
reduction (host wall vs device time), result read-back."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import torch
import paper_2510_19608_b200 as kr
from golden_io import path
case = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c2"
hp = kr.HostProblem(str(path(case, "net.json")), str(path(case, "scen.csv")))
ctx = kr.Context(hp, device=0)
cfg = kr.ReductionConfig(e_bar=3e-3)
ctx.run_reduction(cfg)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0") if "--flush" in sys.argv else None
r = None
for rep in range(4):
    td0 = time.perf_counter(); r = None; td1 = time.perf_counter()
    print(f"previous result free {1e3*(td1-td0):.2f} ms")
    if flush is not None:
        flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ctx.reload(hp); torch.cuda.synchronize(); t1 = time.perf_counter()
    r = ctx.run_reduction(cfg); t2 = time.perf_counter()
    tr0 = time.perf_counter(); _ = r.trace; tr1 = time.perf_counter()
    print(f"trace access {1e3*(tr1-tr0):.2f} ms")
    m = r.model; torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"reload {1e3*(t1-t0):.2f} ms | run wall {1e3*(t2-t1):.2f} ms (device {r.device_ms:.2f}) | model {1e3*(t3-t2):.2f} ms")
