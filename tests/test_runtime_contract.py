"""Runtime contracts of the C ABI beyond single-call parity (GPU).

* Concurrency (operator.hpp:28): an OperatorContext is
  shared read-only and independent solves may run concurrently. Two Python
  threads (the binding releases the GIL) solving on one context give the
  serial results bit for bit.
* Stream ordering at the device edge: a CUDA input still being written by a
  long torch kernel is read only after that kernel, and the returned array is
  ordered before later work on the caller's stream.
* Histories of any length: maxiter = 10**9 allocates nothing maxiter-sized,
  and a 5760-iteration solve (longer than the device history ring) returns
  every entry, bit-identical to the CPU oracle.
"""
import threading

import numpy as np
import pytest

from oracle.oracle import Oracle, Problem

pytestmark = pytest.mark.gpu


def _ctx(acg, prob, math="exact"):
    g = acg.vertical_grid(prob.n_z, prob.h)
    pan = acg.cubed_sphere_panel(prob.m) if prob.sphere else acg.planar_panel(prob.m, prob.extent)
    return acg.OperatorContext(acg.vertical_profile(g, prob.omega2, prob.lambda2), pan, math=math)


def test_two_threads_one_context_bit_identical(acg):
    prob = Problem(96, 48)
    ctx = _ctx(acg, prob)
    fs = [acg.random_field(prob.m, prob.n_z, s) for s in (42, 7, 11, 13)]
    serial = [acg.solve(ctx, f, epsilon=1e-9, maxiter=400) for f in fs]
    out = [[None] * len(fs) for _ in range(2)]
    errs = []

    def work(t):
        try:
            for rep in range(3):
                for a, f in enumerate(fs):
                    out[t][a] = acg.solve(ctx, f, epsilon=1e-9, maxiter=400)
                    # interleave the other entry points too
                    acg.apply(ctx, f)
                    acg.true_residual(ctx, out[t][a][0], f)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for t in range(2):
        for (u, r), (us, rs) in zip(out[t], serial):
            assert r.iterations == rs.iterations
            assert np.array_equal(r.residual_history, rs.residual_history)
            assert np.array_equal(u, us)


def test_device_input_from_a_pending_torch_kernel(acg):
    torch = pytest.importorskip("torch")
    prob = Problem(64, 32)
    ctx = _ctx(acg, prob)
    host = acg.random_field(prob.m, prob.n_z, 42)
    u_ref, r_ref = acg.solve(ctx, host, epsilon=1e-10, maxiter=300)
    src = torch.from_numpy(host).cuda()
    torch.cuda.synchronize()
    for _ in range(3):
        f = torch.zeros_like(src)
        torch.cuda._sleep(50_000_000)  # ~25 ms of device time on the current stream
        f.copy_(src)                   # the input is complete only after the sleep
        u, r = acg.solve(ctx, f, epsilon=1e-10, maxiter=300)
        s = (u * 1.0).cpu().numpy()    # consumed on the caller's stream right away
        assert r.iterations == r_ref.iterations
        assert np.array_equal(r.residual_history, r_ref.residual_history)
        assert np.array_equal(s, u_ref)
    # output buffer reuse: a freed block handed back by torch's allocator
    x = torch.from_numpy(acg.random_field(prob.m, prob.n_z, 5)).cuda()
    y_ref = acg.apply(ctx, x.cpu().numpy())
    for _ in range(3):
        junk = torch.empty_like(x)
        torch.cuda._sleep(20_000_000)
        junk.fill_(3.0)
        del junk                       # its block may be y's storage below
        y = acg.apply(ctx, x)
        assert np.array_equal(y.cpu().numpy(), y_ref)


def test_unbounded_maxiter(acg):
    prob = Problem(16, 8)
    ctx = _ctx(acg, prob)
    f = acg.random_field(prob.m, prob.n_z, 42)
    u1, r1 = acg.solve(ctx, f, epsilon=1e-10, maxiter=10**9)
    u2, r2 = acg.solve(ctx, f, epsilon=1e-10, maxiter=500)
    assert r1.converged and r1.iterations == r2.iterations
    assert len(r1.residual_history) == r1.iterations + 1
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(u1, u2)


@pytest.mark.parametrize("variant", ["interleaved", "standard"])
def test_history_longer_than_the_device_ring(acg, variant):
    prob = Problem(96, 2, False, 10.0, 100.0)  # 5760 iterations to ||r|| < 1e-300
    ctx = _ctx(acg, prob)
    o = Oracle(prob)
    f = o.random_field(42)
    kw = dict(epsilon=1e-300, tau=1e-300, maxiter=6000, variant=variant)
    u, r = acg.solve(ctx, f, **kw)
    uo, ro = o.solve(f, **kw)
    assert r.iterations == ro.iterations > 4096
    for h in ("residual_history", "kappa_history", "alpha_history", "beta_history"):
        assert np.array_equal(getattr(r, h), getattr(ro, h)), h
    assert np.array_equal(u, uo)


def test_context_destroyed_before_its_fields(acg):
    """A garbage collector may finalise an OperatorContext before the capi fields
    and solvers created on it: destroying the context frees their device memory
    and orphans the handles, later destroys only free the handles, and other
    calls on them raise instead of touching freed memory."""
    import gc
    from paper_1302_7193_b200 import capi
    prob = Problem(16, 8)
    ctx = _ctx(acg, prob)
    view = capi.Context.borrow(ctx._handle)  # no owner reference: the context may go first
    f = view.field().fill_random(1)
    s = capi.Solver(view, maxiter=5)
    s.start(f)
    del ctx
    gc.collect()
    with pytest.raises(ValueError):
        f.download()
    with pytest.raises(ValueError):
        s.iterate(1)
    s.close()
    f.close()
    view.h = None  # the borrowed handle is gone with its owner


def test_step_api_histories_longer_than_the_ring(acg):
    """The step API (acg_solver_iterate, what bench.py drives) drains the history
    rings itself: 6000 iterations in two calls return every entry."""
    from paper_1302_7193_b200 import capi
    prob = Problem(96, 2, False, 10.0, 100.0)  # 5760 iterations to ||r|| < 1e-300
    o = Oracle(prob)
    ctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag)
    f = ctx.field().upload(o.random_field(42))
    s = capi.Solver(ctx, epsilon=1e-300, tau=1e-300, maxiter=6000)
    s.start(f)
    s.iterate(3000)
    s.iterate(3000)
    r = s.finish()
    uo, ro = o.solve(o.random_field(42), epsilon=1e-300, tau=1e-300, maxiter=6000)
    assert r["iterations"] == ro.iterations > 4096
    for h in ("residual_history", "kappa_history", "alpha_history", "beta_history"):
        assert np.array_equal(r[h], getattr(ro, h)), h
    s.close()
    f.close()
    ctx.close()
