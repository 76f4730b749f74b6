import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1302_7193_b200 import capi
import paper_1302_7193_b200 as acg
for cfg in [(1024, 128), (512, 128)]:
    m, n_z = cfg
    g = acg.vertical_grid(n_z, 1e-2)
    ctx0 = acg.OperatorContext(acg.vertical_profile(g, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(m))
    ctx = capi.Context.borrow(ctx0._handle, ctx0)
    f = ctx.field().fill_random(42)
    s = capi.Solver(ctx, epsilon=1e-300, tau=1e-300, maxiter=20000)
    s.start(f)
    for chunk in range(20):
        s.iterate(500)
        st = s.state() if hasattr(s, "state") else None
    r = s.finish()
    print(cfg, "iterations", r["iterations"], "converged", r["converged"], "last residual", r["residual_history"][-1])
