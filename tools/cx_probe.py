import os, sys
sys.path[:0] = ['.', 'tests']
import paper_2510_19608_b200 as kr
from golden_io import path
for case in ['c2']:
    ctx = kr.Context(kr.HostProblem(str(path(case, 'net.json')), str(path(case, 'scen.csv'))))
    try:
        r = ctx.run_reduction(kr.ReductionConfig(e_bar=3e-3, objective='complex'))
        print(case, os.environ.get('KRONRED_CPLX_K'), 'ok', len(r.trace), r.device_ms, ctx.last_run_device_loop)
    except Exception as e:
        print(case, os.environ.get('KRONRED_CPLX_K'), 'ERR', e)
