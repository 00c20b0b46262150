"""X-parity of a BASELINE config against the oracle's reference-order solution, through
factor products only (sk_solution_stacked_r: streaming TSQR of [V_gpu, V_ref] on the device).

TEST INFRASTRUCTURE (runs the CPU oracle): python tools/xparity_config.py 3 [--threads N]
Config 3 needs ~25 GB of host memory for V_ref (1,048,576 x 2908) and ~6.5 min of oracle
time on 16 threads; the result is recorded in DESIGN.md section 2."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    import numpy as np
    import paper_2605_28274_b200 as sk
    from paper_2605_28274_b200.problems import baseline_config
    from oracle import pyoracle as po
    from make_config_golden import oracle_inputs
    po.use_threads(args.threads)
    method, a, b, c1, c2, max_iter = oracle_inputs(args.config)
    t0 = time.time()
    ref = po.solve(method, a, b, c1, c2, po.Config(eps_tol=1e-8, max_iter=max_iter), po.REFERENCE_ORDER)
    t_oracle = time.time() - t0
    cfg = baseline_config(args.config)
    scfg = sk.SolverConfig(eps_tol=cfg.eps_tol, max_iter=cfg.max_iter)
    lyap = cfg.method == "cg_lyapunov"
    if cfg.method == "cg":
        sol = sk.factorized_cg(cfg.a, cfg.b, cfg.c1, cfg.c2, scfg)
    elif lyap:
        sol = sk.factorized_cg_lyapunov(cfg.a, cfg.c1, scfg)
    else:
        sol = sk.factorized_bicgstab(cfg.a, cfg.b, cfg.c1, cfg.c2, scfg)
    t0 = time.time()
    d, nref = sk.x_distance(sol, ref.V, ref.core, ref.V if lyap else ref.W, lyapunov=lyap)
    out = {"config": f"C{args.config}", "x_parity": d, "x_ref_norm": nref, "gpu_iterations": sol.history.iterations(),
           "ref_iterations": int(ref.n_iterations), "gpu_status": sol.status, "ref_status": ref.status,
           "oracle_s": t_oracle, "x_distance_s": time.time() - t0, "threads": args.threads}
    print(json.dumps(out))
