import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_13624_b200 as B
ctx = B.Context(0)
o = np.zeros(3)
B._check(B.lib().bmpc_debug_latency_probe(ctx._h, B._ptr(o)))
print("LAT dfma, lds, ddiv cycles:", o, flush=True)
print("RIC", B.debug_ric_step_cycles(512, True, ctx), flush=True)
