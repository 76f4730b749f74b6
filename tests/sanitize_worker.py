"""Worker for tests/test_sanitizers.py: small solves through every kernel family
(run under compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck).

Covers the interleaved loop (TMEM Thomas sweep K1 with its cp.async ring and
tcgen05 alloc/dealloc, the pair stencil sweep K2, fused reduction stage 1 +
the wide stage-2 tree with PDL early starts), the standard loop (apply,
precondition, BLAS-1, k_tree1 path), fp32 (k_thomas_tm2 / k_fused_spmv_pair),
FAST math, the host transfers (K7 transposes), the device RNG, and p = 2
virtual slabs (halo copies, slab-sum combine). Checks the results against the
CPU oracle so a sanitizer run is also a parity run.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1302_7193_b200 as acg  # noqa: E402
from oracle.oracle import Oracle, Problem  # noqa: E402

# argv: cases "MxNZ" (fp64 and fp32) or "MxNZ:f64" / "MxNZ:f32"
DTYPES = {"f64": np.float64, "f32": np.float32}


def cases():
    if len(sys.argv) < 2:
        return [(32, 16, None), (256, 6, None)]
    out = []
    for a in sys.argv[1:]:
        shape, _, dt = a.partition(":")
        m, n_z = (int(x) for x in shape.split("x"))
        out.append((m, n_z, DTYPES[dt] if dt else None))
    return out


def main():
    for m, n_z, only in cases():
        prob = Problem(m, n_z)
        o = Oracle(prob)
        g = acg.vertical_grid(n_z, prob.h)
        pro = acg.vertical_profile(g, prob.omega2, prob.lambda2)
        pan = acg.cubed_sphere_panel(m)
        for dt, cls in ((np.float64, acg.OperatorContext), (np.float32, acg.OperatorContextF32)):
            if only is not None and dt != only:
                continue
            for math, slabs in (("exact", 1), ("fast", 1), ("exact", 2)):
                ctx = cls(pro, pan, math=math, slabs=slabs)
                f = o.random_field(42, dt)
                eps = 1e-8 if dt == np.float64 else 1e-4
                for variant in ("interleaved", "standard"):
                    u, r = acg.solve(ctx, f, epsilon=eps, maxiter=40, variant=variant)
                    if math == "exact":
                        uo, ro = o.solve(f, epsilon=eps, maxiter=40, variant=variant)
                        tag = (m, n_z, np.dtype(dt).name, variant, math, slabs)
                        if ctx.info["exact_tree"]:  # slabs are reduction-tree nodes: same bits
                            assert r.iterations == ro.iterations, tag
                            assert np.array_equal(r.residual_history, ro.residual_history), tag
                            assert np.array_equal(u, uo), tag
                        else:  # slab sums combined pairwise: the north-star tolerances
                            tol = 1e-10 if dt == np.float64 else 1e-4
                            n = min(len(r.residual_history), len(ro.residual_history))
                            assert abs(r.iterations - ro.iterations) <= 1, tag
                            assert (np.abs(r.residual_history[:n] - ro.residual_history[:n]).max()
                                    <= tol * ro.residual_history[0]), tag
                if dt == np.float64 and math == "exact":  # the CSR backend (acg_csr.cuh)
                    u, r = acg.solve(ctx, f, epsilon=eps, maxiter=40, variant="standard",
                                     backend="csr")
                x = o.random_field(5, dt)
                y = acg.apply(ctx, x)
                z = acg.precondition(ctx, x)
                acg.true_residual(ctx, x, f)
                if math == "exact":
                    assert np.array_equal(y, o.apply(x)) and np.array_equal(z, o.precondition(x))
                h = acg.apply(ctx, np.ascontiguousarray(np.transpose(x, (1, 2, 0))),
                              layout="horizontal")
                assert np.array_equal(np.transpose(h, (2, 0, 1)), y)
            if only is None or only == np.float64:
                assert np.array_equal(acg.random_field(m, n_z, 42), o.random_field(42))
        print(f"case {m}x{n_z} ok", flush=True)
    if os.environ.get("SANITIZE_ASYNC", "1") != "0":
        async_transfers()
    print("SANITIZE_DONE", flush=True)


def async_transfers():
    """Copy-stream transfers overlapping a solve (upload_async of the next
    right-hand side, download_async of the previous solution), both layouts.
    Columns taller than TMEM holds (k_thomas), so synccheck can run it too."""
    from paper_1302_7193_b200 import capi
    nz = 272
    prob = Problem(32, nz)
    o = Oracle(prob)
    ctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag)
    shape = (32, 32, nz)
    hf = [capi.HostBuffer(shape) for _ in range(2)]
    hu = [capi.HostBuffer(shape) for _ in range(2)]
    for i, h in enumerate(hf):
        h.array[...] = o.random_field(40 + i)
    fs, us = [ctx.field(), ctx.field()], [ctx.field(), ctx.field()]
    fs[0].upload_async(hf[0].array)
    for i in range(2):
        if i == 0:
            fs[1].upload_async(hf[1].array, layout=capi.VERTICAL)
        capi.solve(ctx, fs[i], u_out=us[i], epsilon=1e-9, maxiter=60)
        us[i].download_async(hu[i].array)
    for i in range(2):
        us[i].wait()
        uo, _ = o.solve(hf[i].array.copy(), epsilon=1e-9, maxiter=60)
        assert np.array_equal(hu[i].array, uo)
    h2 = capi.HostBuffer((32, nz, 32))
    us[0].download_async(h2.array, layout=capi.HORIZONTAL)
    us[0].wait()
    assert np.array_equal(h2.array, np.ascontiguousarray(hu[0].array.transpose(1, 2, 0)))
    for x in fs + us + hf + hu + [h2]:
        x.close()
    ctx.close()
    print("async transfers ok", flush=True)


if __name__ == "__main__":
    main()
