# S3_TIMING variant: per-phase scorer clocks at iterations 1/100/500/850, S forced
for S in 1 2 4; do
  echo "== S=$S"
  KRONRED_S3_S=$S KRONRED_LIB=tools/_var_timing/libkronred_b200.so timeout 120 python -c "
import sys; sys.path[:0]=['.','tests']
import paper_2510_19608_b200 as kr
from golden_io import path
ctx=kr.Context(kr.HostProblem(str(path('c2','net.json')),str(path('c2','scen.csv'))),device=0)
ctx.run_reduction(kr.ReductionConfig(e_bar=3e-3))
" 2>&1 | sort | uniq | head -40
done
