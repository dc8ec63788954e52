import sys, os, json, subprocess
for c in sys.argv[1:]:
    code = f"""
import sys; sys.path.insert(0, 'bisect/{c}')
import numpy as np
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import acr_solve
from paper_1604_00617_b200.system import Tolerance
cc = P.CONFIGS['cfg4']
u, rep = acr_solve(P.make_config('cfg4'), Tolerance(cc['eps']), leaf_size=cc['leaf'])
print('{c}', rep.residual, rep.reduce_ms, rep.max_rank)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
