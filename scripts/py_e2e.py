"""End-to-end time of the reference-facing Python call at C3: anisocg.solve(ctx, numpy f)
(pageable host arrays through the host shim) against the device-resident loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import anisocg as acg

m, n_z, it = 1024, 128, 100
g = acg.vertical_grid(n_z, 1e-2)
ctx = acg.OperatorContext(acg.vertical_profile(g, 6.71e-4, 3.32e-2), acg.cubed_sphere_panel(m))
f = acg.random_field(m, n_z, 42)
for rep in range(3):
    t0 = time.perf_counter()
    u, r = acg.solve(ctx, f, epsilon=1e-300, tau=1e-300, maxiter=it)
    dt = time.perf_counter() - t0
    t = r.timings
    print(f"anisocg.solve numpy: {dt*1e3:.1f} ms for {it} iterations -> {it/dt:.1f} it/s "
          f"(loop+init {t.total_s*1e3:.1f} ms)", flush=True)
