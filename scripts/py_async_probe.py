"""Where does the e2e stream lose time? Solve alone vs with a concurrent
async upload / download of another field (C3 fp64, 100 iterations)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_7193_b200 import capi  # noqa: E402
import paper_1302_7193_b200 as acg  # noqa: E402

m, n_z, it = 1024, 128, 100
gr = acg.vertical_grid(n_z, 1e-2)
ctx0 = acg.OperatorContext(acg.vertical_profile(gr, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(m))
ctx = capi.Context.borrow(ctx0._handle, ctx0)
f = ctx.field().fill_random(42)
u = ctx.field()
x = ctx.field().fill_random(3)
hb = capi.HostBuffer((m, m, n_z), np.float64)
hb2 = capi.HostBuffer((m, m, n_z), np.float64)
x.download(out=hb.array)
kw = dict(epsilon=1e-300, tau=1e-300, maxiter=it)
capi.solve(ctx, f, u_out=u, **kw)


def t_solve():
    t = time.perf_counter()
    capi.solve(ctx, f, u_out=u, **kw)
    return (time.perf_counter() - t) * 1e3


for rep in range(2):
    print("solve alone          ", [round(t_solve(), 1) for _ in range(3)])
    res = []
    for _ in range(3):
        x.upload_async(hb.array)
        res.append(round(t_solve(), 1))
        x.wait()
    print("solve + upload_async ", res)
    res = []
    for _ in range(3):
        x.download_async(hb2.array)
        res.append(round(t_solve(), 1))
        x.wait()
    print("solve + download_async", res)
    res = []
    for _ in range(3):
        x.upload_async(hb.array)
        x.download_async(hb2.array)
        res.append(round(t_solve(), 1))
        x.wait()
    print("solve + both          ", res)
    t = time.perf_counter(); x.upload_async(hb.array); x.wait(); a = time.perf_counter() - t
    t = time.perf_counter(); x.download_async(hb2.array); x.wait(); b = time.perf_counter() - t
    print(f"upload_async alone {a*1e3:.1f} ms, download_async alone {b*1e3:.1f} ms")
