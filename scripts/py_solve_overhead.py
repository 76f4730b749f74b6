import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1302_7193_b200 import capi
import paper_1302_7193_b200 as acg
m, n_z = 1024, 128
gr = acg.vertical_grid(n_z, 1e-2)
ctx0 = acg.OperatorContext(acg.vertical_profile(gr, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(m))
ctx = capi.Context.borrow(ctx0._handle, ctx0)
f = ctx.field().fill_random(42); u = ctx.field()
for it in (1, 100):
    for rep in range(3):
        t = time.perf_counter()
        r = capi.solve(ctx, f, u_out=u, epsilon=1e-300, tau=1e-300, maxiter=it)
        w = time.perf_counter() - t
        print(it, f"wall {w*1e3:.1f} ms", {k: round(v*1e3, 2) for k, v in r["timings"].items()} if isinstance(r.get("timings"), dict) else r.get("timings"))
