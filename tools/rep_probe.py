"""Timing probe: repeated runs on one context, and fresh contexts (host wall)."""
import sys, time
sys.path[:0] = ['/root/repo', '/root/repo/tests']
import paper_2510_19608_b200 as kr
from golden_io import path
import torch
hp = kr.HostProblem(str(path("c2", "net.json")), str(path("c2", "scen.csv")))
cfg = kr.ReductionConfig(e_bar=3e-3)
ctx = kr.Context(hp, device=0)
for i in range(3):
    r = ctx.run_reduction(cfg); print("same ctx", i, round(r.device_ms, 1))
for i in range(3):
    t0 = time.perf_counter(); c = kr.Context(hp, device=0); t1 = time.perf_counter()
    r = c.run_reduction(cfg); t2 = time.perf_counter()
    del c; torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"fresh ctx {i}: create {1e3*(t1-t0):.1f} ms, run wall {1e3*(t2-t1):.1f} ms (device {r.device_ms:.1f}), destroy {1e3*(t3-t2):.1f}")
