import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_1302_7193_b200 import capi
from oracle.oracle import Oracle, Problem
o = Oracle(Problem(32, 16))
ctx = capi.Context(o.ap, o.bp, o.cp, o.d, o.area, o.east, o.north, o.diag)
y = ctx.field().upload(o.random_field(3)); x = ctx.field()
capi.precondition(ctx, y, x)
print("precondition ok", np.array_equal(x.download(), o.precondition(o.random_field(3))))
