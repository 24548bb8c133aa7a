"""Full-length golden runs of the UNMODIFIED reference solver (oracle/_ref,
built by oracle/Makefile from /root/reference/proj/include) at BASELINE.json's
north-star sizes. Test infrastructure only.

    python tests/golden/make_fullrun.py c3      # 4096^2, 50 iterations
    python tests/golden/make_fullrun.py c4      # 384^3, 30 iterations
    python tests/golden/make_fullrun.py c2      # 1024^2 until |d dual| < 1e-6
    python tests/golden/make_fullrun.py c1      # 256^2, 100 iterations

The inputs come from the library's shared generator
(bfm_synthetic_densities); their SHA-256 is stored so a replay
on other inputs fails loudly. Per iteration the reference's Solver::step()
(solver.hpp:286-310) is driven exactly like tests/test_gpu_fullrun.py drives
the GPU solver, and we record:
  * the full IterationStats (solver.hpp:78-88) and Solver::sigma();
  * SHA-256 of the raw bits of phi and psi (the fields are 128-432 MiB, too
    large to commit) plus 1024 sampled values of each (fixed node indices), so
    a mismatch can be sized without the reference present;
then Solver::run() (rule loop, solver.hpp:211-226) with max_iterations equal
to the steps taken, which finishes immediately (the iteration cap is the first
rule that fires) and returns the gauge-fixed report (finish, :330-349): its
phi/psi/map hashes and samples, dual, primal, residual, termination.

The fields themselves never leave this container; the GPU box compares hashes.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402
import paper_1905_12154_b200 as bfm  # noqa: E402
from paper_1905_12154_b200 import synthetic  # noqa: E402

# (generator config, n, seed, steps or None = until |d dual| < 1e-6, cap)
RUNS = {
    "c1": (1, 256, 1, 100, None),
    "c2": (2, 1024, 2, None, 1000),
    "c3": (3, 4096, 3, 50, None),
    "c4": (4, 384, 4, 30, None),
}
STAT_FIELDS = ("iteration", "residual", "dual_value", "sigma_first", "sigma_second",
               "grad_norm_sq_first", "grad_norm_sq_second", "increase_first", "increase_second")
NSAMPLE = 1024


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sample_index(size: int) -> np.ndarray:
    return np.sort(np.random.default_rng(12154).choice(size, size=min(NSAMPLE, size), replace=False))


def path_for(name: str) -> str:
    return os.path.join(HERE, f"fullrun_{name}.npz")


def inputs(name: str):
    config, n, seed, _, _ = RUNS[name]
    return synthetic._shared(config, n, seed)


def main(name: str) -> None:
    config, n, seed, steps, cap = RUNS[name]
    mu, nu = inputs(name)
    idx = sample_index(mu.size)
    max_it = steps if steps is not None else cap
    cfg = bfm.SolverConfig(tolerance=-1.0, max_iterations=max_it)
    s = O.RefSolver(mu, nu, cfg)
    trace, sig, phi_h, psi_h, phi_s, psi_s, secs = [], [], [], [], [], [], []
    prev = 0.0  # trace[0] is compared with the initial pair value 0
    k = 0
    while k < max_it:
        t0 = time.perf_counter()
        st = s.step()
        secs.append(time.perf_counter() - t0)
        k += 1
        phi, psi = s.phi(), s.psi()
        trace.append([getattr(st, f) for f in STAT_FIELDS])
        sig.append(s.sigma())
        phi_h.append(sha(phi))
        psi_h.append(sha(psi))
        phi_s.append(phi.reshape(-1)[idx])
        psi_s.append(psi.reshape(-1)[idx])
        print(f"{name} it {k}: dual {st.dual_value!r} sigma {s.sigma()!r} ({secs[-1]:.1f} s)",
              flush=True)
        if steps is None and abs(st.dual_value - prev) < 1e-6:
            break
        prev = st.dual_value
    if k != max_it:
        # stopped early (C2's |d dual| rule): replay the k steps on a solver
        # capped at k so that run() finishes at once, as below
        s = O.RefSolver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=k))
        for _ in range(k):
            s.step()
    # the rule loop with the cap at the steps taken: the cap is the first rule
    # that fires, so run() only does finish() (probe, gauge fix, map, primal)
    s2cfg_note = "run() after the steps with max_iterations == steps taken"
    rep = s.run()
    out = dict(
        name=np.array(name), generator=np.array([config, n, seed]), steps=np.array(k),
        mu_sha=np.array(sha(mu)), nu_sha=np.array(sha(nu)), sample_index=idx,
        trace=np.array(trace), stat_fields=np.array(STAT_FIELDS), sigma=np.array(sig),
        phi_sha=np.array(phi_h), psi_sha=np.array(psi_h),
        phi_sample=np.array(phi_s), psi_sample=np.array(psi_s), step_seconds=np.array(secs),
        threads=np.array(os.cpu_count()), note=np.array(s2cfg_note),
        rep_scalars=np.array([rep.iterations, rep.dual_value, rep.primal_cost, rep.residual]),
        rep_termination=np.array(rep.termination),
        rep_phi_sha=np.array(sha(rep.phi)), rep_psi_sha=np.array(sha(rep.psi)),
        rep_map_sha=np.array([sha(m) for m in rep.map]),
        rep_phi_sample=rep.phi.reshape(-1)[idx], rep_psi_sample=rep.psi.reshape(-1)[idx],
        rep_map_sample=np.array([m.reshape(-1)[idx] for m in rep.map]),
        rep_trace_len=np.array(len(rep.trace)),
    )
    np.savez_compressed(path_for(name), **out)
    print(f"wrote {path_for(name)}: {k} steps, dual {rep.dual_value!r}, "
          f"{sum(secs):.0f} s of reference steps")


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c1"]:
        main(nm)
