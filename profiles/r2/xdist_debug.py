import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2605_28274_b200 as sk
from paper_2605_28274_b200 import problems as pr
g = int(sys.argv[1]); iters = int(sys.argv[2])
a = pr.laplacian_2d(g)
c1 = pr.random_rhs(g * g, 1, 1234)
sol = sk.factorized_cg_lyapunov(a, c1, sk.SolverConfig(eps_tol=1e-30, max_iter=iters))
print("solved", sol.status, sol.rv, flush=True)
v = sol.V
print("V copied", v.shape, flush=True)
t0 = time.time()
d, nref = sk.x_distance(sol, v, sol.core, v, lyapunov=True)
print("self distance", d, nref, time.time() - t0)
