import sys, numpy as np
sys.path.insert(0, ".")
import paper_2605_28274_b200 as sk
from paper_2605_28274_b200.problems import baseline_config
g = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
from paper_2605_28274_b200 import problems as pr
a = pr.laplacian_2d(g)
c1 = pr.random_rhs(g * g, 1, 1234)
hs = []
for rep in range(3):
    sol = sk.factorized_cg_lyapunov(a, c1, sk.SolverConfig(eps_tol=1e-8, max_iter=int(sys.argv[3]) if len(sys.argv) > 3 else 300))
    hs.append(sol.history.rel_residuals().copy())
    print('paths', sol.stats['paths'], 'iters', sol.history.iterations(), 'launches', sol.stats['kernel_launches'])
    sol.free()
np.save(sys.argv[1], np.array(hs))
print("status", sol.status, "len", len(hs[0]), "repeatable", all(np.array_equal(hs[0], h) for h in hs))
