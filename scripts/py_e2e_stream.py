"""The bench's e2e stream (4 solves, async transfers on the copy stream) repeated,
with per-solve times, to see its spread (C3 fp64, 100 iterations per solve)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_7193_b200 import capi  # noqa: E402
import paper_1302_7193_b200 as acg  # noqa: E402

m, n_z, it, ns = 1024, 128, 100, 4
g = acg.vertical_grid(n_z, 1e-2)
ctx0 = acg.OperatorContext(acg.vertical_profile(g, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(m))
ctx = capi.Context.borrow(ctx0._handle, ctx0)
hf = [capi.HostBuffer((m, m, n_z)) for _ in range(2)]
hu = [capi.HostBuffer((m, m, n_z)) for _ in range(2)]
src = ctx.field().fill_random(42)
src.download(out=hf[0].array)
hf[1].array[...] = hf[0].array
fs, us = [ctx.field(), ctx.field()], [ctx.field(), ctx.field()]
kw = dict(epsilon=1e-300, tau=1e-300, maxiter=it)
fs[0].upload(hf[0].array)
capi.solve(ctx, fs[0], u_out=us[0], **kw)
for rep in range(int(os.environ.get("REPS", "6"))):
    t0 = time.perf_counter()
    marks = []
    fs[0].upload_async(hf[0].array)
    for i in range(ns):
        if i + 1 < ns:
            fs[(i + 1) % 2].upload_async(hf[(i + 1) % 2].array)
        t = time.perf_counter()
        capi.solve(ctx, fs[i % 2], u_out=us[i % 2], **kw)
        marks.append(round((time.perf_counter() - t) * 1e3, 1))
        us[i % 2].download_async(hu[i % 2].array)
    for u in us:
        u.wait()
    wall = time.perf_counter() - t0
    print(f"stream: {ns * it / wall:.1f} it/s, wall {wall * 1e3:.0f} ms, solves {marks}", flush=True)
