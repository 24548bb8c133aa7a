"""Ad-hoc GPU diagnostics (not collected by pytest)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from fractions import Fraction as F
import numpy as np
import oracle_lib as O
import paper_1905_12154_b200 as bfm
from paper_1905_12154_b200 import synthetic

def exact_ct(phi):
    shape = phi.shape
    coords = [bfm.axis_coords(n) for n in shape]
    out = np.empty(shape)
    idx = list(np.ndindex(*shape))
    for k in idx:
        best = None
        for j in idx:
            v = F(-phi[j])
            for a in range(len(shape)):
                x, y = coords[a][k[a]], coords[a][j[a]]
                v += F(0.5 * x * x) + F(0.5 * y * y) - F(x) * F(y)
            if best is None or v < best: best = v
        out[k] = float(best)  # nearest; compare separately
        d = float(best)
        if F(d) > best: d = np.nextafter(d, -np.inf)
        out[k] = d if d != 0 else 0.0
    return out

rng = np.random.default_rng(0)
for shape in [(3,), (5,), (6,), (7,), (12,), (3, 5), (2, 3, 2), (5, 3), (6, 10)]:
    for kind in range(2):
        phi = rng.uniform(-1, 1, shape)
        g = bfm.ctransform(phi)
        r = O.orc_ctransform(phi)
        e = exact_ct(phi)
        nb = O.n_bit_diff(g, r)
        print(shape, kind, "gpu!=orc", nb, "orc!=exact", O.n_bit_diff(r, e), "gpu!=exact", O.n_bit_diff(g, e))
        if nb:
            bad = np.argwhere(O.bits(g) != O.bits(r))[:3]
            for b in bad:
                b = tuple(b)
                print("   ", b, g[b].hex(), r[b].hex())
# solver: un-gauged fields after 1..3 steps vs restatement
for shape_fn in [lambda: synthetic.c1(32), lambda: synthetic.c1(64)]:
    mu, nu = shape_fn()
    s = bfm.Solver(mu, nu, bfm.SolverConfig(tolerance=-1.0, max_iterations=10))
    for it in range(1, 4):
        st = s.step()
        phi_o, psi_o, duals = O.orc_run_steps(mu, nu, it)
        print("solver", mu.shape, it, "phi diff", O.n_bit_diff(s.phi(), phi_o), "psi diff", O.n_bit_diff(s.psi(), psi_o),
              "dual", st.dual_value, duals[-1])
