"""Generate tests/golden/csr_golden.npz from the REFERENCE's CsrBackend.

backend = "csr" (solver.hpp:126-145: assemble_csr + spmv_csr + the stored
tridiagonal solve, csr.hpp:92-221) driven by pcg_standard, run by the
unmodified reference compiled in oracle/_ref. The CSR summation order follows
the fields' layout, so both layouts are recorded.

    python tests/golden/make_csr_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Problem, Reference  # noqa: E402

CASES = [  # tag, problem, dtype, solve kwargs
    ("s8_16", Problem(8, 16), np.float64, dict(epsilon=1e-8, maxiter=300)),
    ("p13_7", Problem(13, 7, False), np.float64, dict(epsilon=1e-10, maxiter=300)),
    ("s32_24_f32", Problem(32, 24), np.float32, dict(epsilon=1e-4, maxiter=300)),
    ("s64_32_fix", Problem(64, 32), np.float64, dict(epsilon=1e-300, tau=1e-300, maxiter=25)),
]


def main():
    out = {}
    for tag, prob, dt, kw in CASES:
        ref = Reference(prob)
        for layout in (0, 1):
            f = ref.random_field(42, dt, layout)
            u, r = ref.solve(f, variant="standard", backend="csr", layout=layout, **kw)
            key = f"{tag}_L{layout}"
            out[f"{key}_u"] = u
            out[f"{key}_res"], out[f"{key}_kap"] = r.residual_history, r.kappa_history
            out[f"{key}_alp"], out[f"{key}_bet"] = r.alpha_history, r.beta_history
            out[f"{key}_meta"] = np.array([r.iterations, int(r.converged), r.true_residual])
            print(key, r.iterations, r.converged)
    np.savez_compressed(os.path.join(HERE, "csr_golden.npz"), **out)


if __name__ == "__main__":
    main()
