"""Regenerates the committed golden fixtures under tests/golden/.

rng_golden.json  -- std::mt19937_64 / uniform_real_distribution / Box-Muller values
                    from a g++-compiled program (oracle/gen_rng_golden.cpp), pinning
                    the oracle's C restatement of the reference generators.
histories.json   -- per-iteration relative residual histories of the oracle
                    (both arithmetic modes) on the small BASELINE configs and the
                    reference's own test instances; the GPU tests compare against
                    these without needing /root/reference on the box.

Run from the repo root: python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))


def rng():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "gen")
        subprocess.check_call(["g++", "-O2", "-std=c++17", os.path.join(ROOT, "oracle", "gen_rng_golden.cpp"),
                               "-o", exe])
        out = subprocess.check_output([exe]).decode()
    data = json.loads(out)
    with open(os.path.join(HERE, "rng_golden.json"), "w") as f:
        json.dump(data, f, indent=1)


def histories():
    import numpy as np
    from oracle import pyoracle as po
    out = {}
    a = po.laplacian_2d(64)
    c1 = po.random_rhs(4096, 1, 1234)
    c1 /= np.linalg.norm(c1)
    c2 = po.random_rhs(4096, 1, 1235)
    c2 /= np.linalg.norm(c2)
    cfg = po.Config(eps_tol=1e-8, max_iter=500)
    for mode, name in [(po.REPRODUCIBLE, "reproducible"), (po.REFERENCE_ORDER, "reference_order")]:
        s = po.factorized_cg(a, a, c1, c2, cfg, mode)
        out[f"config1_cg_{name}"] = {"status": s.status, "rel_residual": [float(x) for x in s.rel_residual],
                                     "core_fro": float(np.linalg.norm(s.core))}
    a30 = po.laplacian_2d(30)
    d1 = po.random_rhs(900, 3, 101)
    for mode, name in [(po.REPRODUCIBLE, "reproducible"), (po.REFERENCE_ORDER, "reference_order")]:
        s = po.factorized_cg_lyapunov(a30, d1, po.Config(eps_tol=1e-13, max_iter=25), mode)
        out[f"lyap30_s3_{name}"] = {"status": s.status, "rel_residual": [float(x) for x in s.rel_residual]}
    with open(os.path.join(HERE, "histories.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    rng()
    histories()
    print("golden fixtures written")
