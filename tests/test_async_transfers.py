"""Asynchronous host transfers (acg_field_upload_async / _download_async /
acg_field_wait): the DMA and relayout run on the context's copy stream while
the solver's kernels run; every entry point orders its work after a field's
pending transfer. The results must be exactly those of the synchronous calls.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, Problem

pytestmark = pytest.mark.gpu


def _ctx(capi, prob, slabs=1):
    o = Oracle(prob)
    return o, capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag, slabs=slabs)


@pytest.mark.parametrize("slabs", [1, 2])
def test_round_trip_layouts(slabs):
    from paper_1302_7193_b200 import capi
    o, ctx = _ctx(capi, Problem(64, 24), slabs)
    for layout in (capi.VERTICAL, capi.HORIZONTAL):
        f = ctx.field()
        shape = f._shape(layout, capi.HOST_FULL)
        src = capi.HostBuffer(shape, np.float64)
        dst = capi.HostBuffer(shape, np.float64)
        src.array[...] = np.random.default_rng(3).standard_normal(shape)
        f.upload_async(src.array, layout=layout)
        f.download_async(dst.array, layout=layout)  # same copy stream, after the upload
        f.wait()
        assert np.array_equal(dst.array, src.array)
        # the synchronous download sees the async upload too
        assert np.array_equal(f.download(layout=layout), src.array)
        for x in (f, src, dst):
            x.close()
    ctx.close()


def test_pipelined_solves_equal_serial():
    """Three solves with different right-hand sides, each f uploaded while the
    previous solve runs and each u downloaded while the next one runs, give
    the serial results bit for bit (and the oracle's)."""
    from paper_1302_7193_b200 import capi
    prob = Problem(128, 32)
    o, ctx = _ctx(capi, prob)
    kw = dict(epsilon=1e-10, maxiter=200)
    rhs = [o.random_field(s) for s in (42, 7, 11)]
    serial = [o.solve(f, **kw) for f in rhs]
    hf = [capi.HostBuffer(rhs[0].shape, np.float64) for _ in range(2)]
    hu = [capi.HostBuffer(rhs[0].shape, np.float64) for _ in range(2)]
    fs, us = [ctx.field(), ctx.field()], [ctx.field(), ctx.field()]
    got = []
    hf[0].array[...] = rhs[0]
    fs[0].upload_async(hf[0].array)
    for i in range(3):
        if i + 1 < 3:
            fs[(i + 1) % 2].wait()  # its previous upload is done before hf is rewritten
            hf[(i + 1) % 2].array[...] = rhs[i + 1]
            fs[(i + 1) % 2].upload_async(hf[(i + 1) % 2].array)
        r = capi.solve(ctx, fs[i % 2], u_out=us[i % 2], **kw)
        if i >= 1:  # the previous download is complete: collect it
            us[(i - 1) % 2].wait()
            got.append(hu[(i - 1) % 2].array.copy())
        us[i % 2].download_async(hu[i % 2].array)
        assert r["iterations"] == serial[i][1].iterations
        assert np.array_equal(r["residual_history"], serial[i][1].residual_history)
    us[2 % 2].wait()
    got.append(hu[2 % 2].array.copy())
    for (uo, _), u in zip(serial, got):
        assert np.array_equal(u, uo)
    for x in fs + us + hf + hu:
        x.close()
    ctx.close()


def test_entry_points_order_after_pending_upload():
    """apply right after upload_async reads the uploaded field, not its old
    contents; a field overwritten by a solve waits for its pending download."""
    from paper_1302_7193_b200 import capi
    prob = Problem(96, 40)
    o, ctx = _ctx(capi, prob)
    x_host = o.random_field(5)
    hb = capi.HostBuffer(x_host.shape, np.float64)
    hb.array[...] = x_host
    x, y = ctx.field().fill(0.0), ctx.field()
    for _ in range(3):
        x.fill(0.0)
        x.upload_async(hb.array)
        capi.apply(ctx, x, y)
        assert np.array_equal(y.download(), o.apply(x_host))
    # download_async of u, then a solve that overwrites u: the download holds
    # the old contents
    f = ctx.field().upload(o.random_field(42))
    u = ctx.field().upload(x_host)
    out = capi.HostBuffer(x_host.shape, np.float64)
    u.download_async(out.array)
    capi.solve(ctx, f, u_out=u, epsilon=1e-8, maxiter=50)
    u.wait()
    assert np.array_equal(out.array, x_host)
    for v in (hb, x, y, f, u, out):
        v.close()
    ctx.close()


def test_pageable_host_buffer_rejected():
    from paper_1302_7193_b200 import capi
    prob = Problem(32, 8)
    o, ctx = _ctx(capi, prob)
    f = ctx.field()
    with pytest.raises(Exception, match="page-locked"):
        f.upload_async(np.zeros((32, 32, 8)))
    f.close()
    ctx.close()


def test_async_edges():
    """wait() without transfers returns at once; shape and dtype are checked
    before anything is enqueued; release_scratch frees the staging and the
    next transfer allocates it again; a field destroyed with a transfer in
    flight waits for it."""
    from paper_1302_7193_b200 import capi
    prob = Problem(48, 10)
    o, ctx = _ctx(capi, prob)
    f = ctx.field()
    f.wait()
    hb = capi.HostBuffer((48, 48, 10), np.float64)
    hb.array[...] = o.random_field(3)
    with pytest.raises(ValueError):
        f.upload_async(capi.HostBuffer((48, 10, 48), np.float64).array)
    with pytest.raises(ValueError):
        f.download_async(np.zeros((48, 48, 10), dtype=np.float32))
    f.upload_async(hb.array)
    ctx.release_scratch()  # synchronises the copy stream, frees the staging
    assert np.array_equal(f.download(), hb.array)
    out = capi.HostBuffer((48, 48, 10), np.float64)
    f.download_async(out.array)  # staging re-created
    f.wait()
    assert np.array_equal(out.array, hb.array)
    g = ctx.field()
    g.upload_async(hb.array)
    g.close()  # waits for its transfer before freeing
    f.close()
    ctx.close()
