"""Generate tests/golden/convergence_golden.npz from the REFERENCE implementation.

Convergence-to-epsilon fixtures at the BASELINE sizes (north_star: "same
iteration count to convergence (±1), residual history within 1e-10 relative in
fp64 (1e-4 in fp32), and final solution within the stated relative tolerance").
The reference (oracle/_ref = proj/include/anisocg/*.hpp + src/grid.cpp +
src/profile.cpp compiled from /root/reference by oracle/Makefile) runs each solve
on all host cores here, once; a C3 solve takes ~5 minutes on 8 cores, too long
to repeat inside the GPU test run, so its outputs travel as fixtures:

  * iterations, converged flag, true residual, all four histories (full);
  * sha256 of u's bytes (the EXACT-mode check is bit-identity of the whole
    field), max|u| and u at 65536 seeded positions (the FAST-mode check,
    max|du|/max|u| like verify.cpp:31-39 field_rel_diff);
  * sha256 of f (the device RNG must reproduce fill_random(seed=42)).

Cases (cubed sphere, omega2 = 6.71e-4, H = 1e-2, RHS seed 42, u0 = 0):
  c2_il   fp64 512^2 x 128,  lambda2 = 3.32e-2, eps = 1e-10 (338 it)
  c2_std  same, variant = "standard"                         (338 it)
  c3_il   fp64 1024^2 x 128, lambda2 = 3.32e-2, eps = 1e-10 (664 it)
  c4_il20 fp32 2048^2 x 128, lambda2 = 100, 20 fixed iterations (eps = tau = 1e-300)

    python tests/golden/make_convergence.py [case ...]
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Problem, Reference  # noqa: E402

OUT = os.path.join(HERE, "convergence_golden.npz")
N_SAMPLE = 65536

CASES = {
    "c2_il": dict(m=512, n_z=128, dtype=np.float64, lambda2=3.32e-2,
                  kw=dict(epsilon=1e-10, maxiter=2000, variant="interleaved")),
    "c2_std": dict(m=512, n_z=128, dtype=np.float64, lambda2=3.32e-2,
                   kw=dict(epsilon=1e-10, maxiter=2000, variant="standard")),
    "c3_il": dict(m=1024, n_z=128, dtype=np.float64, lambda2=3.32e-2,
                  kw=dict(epsilon=1e-10, maxiter=2000, variant="interleaved")),
    "c4_il20": dict(m=2048, n_z=128, dtype=np.float32, lambda2=1.0e2,
                    kw=dict(epsilon=1e-300, tau=1e-300, maxiter=20, variant="interleaved")),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_index(n):
    """The seeded flat positions every consumer samples u at."""
    return np.sort(np.random.default_rng(20260214).choice(n, size=min(N_SAMPLE, n), replace=False))


def main(names):
    out = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        c = CASES[name]
        prob = Problem(c["m"], c["n_z"], True, 6.71e-4, c["lambda2"], 1e-2)
        ref = Reference(prob, workers=os.cpu_count() or 1)
        f = ref.random_field(42, c["dtype"])
        t0 = time.time()
        u, res = ref.solve(f, **c["kw"])
        dt = time.time() - t0
        flat = u.reshape(-1)
        out[f"{name}_f_sha"] = np.array(sha(f))
        out[f"{name}_u_sha"] = np.array(sha(u))
        out[f"{name}_u_max"] = np.array(np.abs(flat).max(), dtype=np.float64)
        out[f"{name}_u_sample"] = flat[sample_index(flat.size)].copy()
        out[f"{name}_res"], out[f"{name}_kap"] = res.residual_history, res.kappa_history
        out[f"{name}_alp"], out[f"{name}_bet"] = res.alpha_history, res.beta_history
        out[f"{name}_meta"] = np.array([res.iterations, int(res.converged), res.true_residual])
        print(f"{name}: {res.iterations} iterations, converged={res.converged}, "
              f"true residual {res.true_residual:.6e}, {dt:.1f} s on {os.cpu_count()} threads",
              flush=True)
        np.savez_compressed(OUT, **out)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
