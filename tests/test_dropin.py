"""The drop-in boundary against the reference's OWN headers.

oracle/build_ref.sh compiles tests/dropin/dropin_caller.cpp -- a caller that includes
proj/include/sylkrylov/*.hpp unchanged and uses the reference's SparseMatrix,
read_matrix_market_sparse, laplacian_2d, random_rhs -- together with
paper_2605_28274_b200/dropin/factorized_solvers_b200.cpp (the product's replacement of
the reference's src/factorized_solvers.cpp) and the reference's own Eigen-free sources.
The CPU test checks the link (the reference's mangled entry points are defined by the
product); the GPU test runs the binary and compares its histories bit for bit with the
Python mirror on the same seeded inputs."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_caller")
HAVE_REF = os.path.isdir("/root/reference/proj/include/sylkrylov")


def ensure_built():
    if HAVE_REF:
        from paper_2605_28274_b200 import build
        build.build()
        subprocess.check_call([os.path.join(ROOT, "oracle", "build_ref.sh")], stdout=subprocess.DEVNULL)
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_caller not built (needs /root/reference to compile)")


def test_dropin_defines_the_reference_entry_points():
    ensure_built()
    syms = subprocess.run(["nm", "-C", "--defined-only", EXE], capture_output=True, text=True, check=True).stdout
    for name in ("sylkrylov::factorized_cg(", "sylkrylov::factorized_cg_lyapunov(", "sylkrylov::factorized_bicgstab(",
                 "sylkrylov::true_residual(", "sylkrylov::true_residual_factors(", "sylkrylov::embed(",
                 "sylkrylov::embed_to(", "sylkrylov::small_sylvester_apply("):
        assert name in syms, name
    # the signatures are the reference's own types (no b200 shim types in the caller)
    assert "sylkrylov::b200::" not in syms
    und = subprocess.run(["nm", "-C", "--undefined-only", EXE], capture_output=True, text=True, check=True).stdout
    assert "sk_factorized_cg" in und and "sylkrylov::read_matrix_market_sparse" in und


def parse(out):
    res = {}
    for line in out.splitlines():
        m = re.match(r"(\w+) history (.*)", line)
        if m:
            res[m.group(1)] = np.array([float(x) for x in m.group(2).split()])
        m = re.match(r"(\w+) status=(\w+) iterations=(\d+) rv=(\d+) rw=(\d+) n=(\d+) m=(\d+) true_residual=(\S+)", line)
        if m:
            res[m.group(1) + "_meta"] = (m.group(2), int(m.group(3)), int(m.group(4)), int(m.group(5)), float(m.group(8)))
    return res


@pytest.mark.gpu
def test_dropin_caller_matches_python_mirror_bitwise(sk, tmp_path):
    ensure_built()
    r = subprocess.run([EXE, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "errors_ok=3" in r.stdout
    assert "nonsymmetric: InvalidMatrixError" in r.stdout
    assert "shape: DimensionError: solver: C1/C2 row counts must match A/B" in r.stdout
    assert "rankdef: RankDeficientStartError" in r.stdout
    assert "image 3 x 3: q00=3 q11=4 q21=1 q02=3" in r.stdout
    got = parse(r.stdout)
    from paper_2605_28274_b200 import problems as pr
    a = pr.laplacian_2d(24)
    c1, c2 = pr.random_rhs(a.n_rows, 2, 1234), pr.random_rhs(a.n_rows, 2, 1235)
    cfg = sk.SolverConfig(eps_tol=1e-8)
    cg = sk.factorized_cg(a, a, c1, c2, cfg)
    ly = sk.factorized_cg_lyapunov(a, c1, cfg)
    ca = pr.convection_diffusion_3d(8, (10.0, 10.0, 10.0))
    d1, d2 = pr.random_rhs(ca.n_rows, 2, 99), pr.random_rhs(ca.n_rows, 2, 100)
    bi = sk.factorized_bicgstab(ca, ca, d1, d2, cfg)
    for name, sol in (("cg", cg), ("lyapunov", ly), ("bicgstab", bi)):
        assert np.array_equal(got[name], sol.history.rel_residuals()), name
        status, its, rv, rw, tr = got[name + "_meta"]
        assert status == sol.status and its == sol.history.iterations()
        assert (rv, rw) == sol.core.shape
        assert tr <= 5e-8
