"""BiCGSTAB parity contract, pinned on the CPU oracle alone.

VERDICT round 1 measured that the REPRODUCIBLE history (which the GPU executes bit for
bit) leaves 1e-10 of the REFERENCE_ORDER history after ~20 iterations on the config-2
operators at grid 32 (cd2, winds (10,10)/(10,-10), s = 4) and suspected CGS2 + CholQR
vs the reference's MGS2 + Householder (block_krylov.cpp:79-93, decompositions.cpp:16-78).
These tests pin what that divergence is:

  * the reference-order run diverges from ITSELF at the same rate when ONE entry of C1
    moves by one ulp (same arithmetic, same MGS2 + Householder): the factorized BiCGSTAB
    recurrence (factorized_solvers.cpp:268-381) amplifies any rounding-level
    perturbation ~10x per two iterations on this nonnormal operator pair, so no
    implementation that is not bit-identical to the reference binary (Eigen's own
    summation orders included, which nothing pins -- SURVEY 8c) can hold 1e-10 past the
    leading window;
  * inside the window (the first 16 iterations here) the two modes agree to 1e-10;
  * the contract mode's distance from the reference order stays within a small factor of
    the reference order's own 1-ulp sensitivity at every iteration of the window;
  * both modes converge, with iteration counts within the 1-ulp sensitivity (+-2), and
    both solutions have a true residual at the tolerance.
"""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def runs(po):
    g = 32
    a = po.convection_diffusion_2d(g, (10.0, 10.0))
    b = po.convection_diffusion_2d(g, (10.0, -10.0))
    c1 = po.random_rhs(g * g, 4, 1234)
    c2 = po.random_rhs(g * g, 4, 1235)
    c1p = c1.copy()
    c1p[5, 0] = np.nextafter(c1p[5, 0], np.inf)
    cfg = po.Config(eps_tol=1e-8)
    out = {
        "ref": po.solve(po.BICGSTAB, a, b, c1, c2, cfg, po.REFERENCE_ORDER),
        "ref_ulp": po.solve(po.BICGSTAB, a, b, c1p, c2, cfg, po.REFERENCE_ORDER),
        "rep": po.solve(po.BICGSTAB, a, b, c1, c2, cfg, po.REPRODUCIBLE),
        "ops": (a, b, c1, c2),
    }
    return out


def rel(x, y):
    n = min(len(x), len(y))
    x, y = np.asarray(x[:n]), np.asarray(y[:n])
    return np.abs(x - y) / np.abs(y)


def test_reference_order_is_not_self_consistent_to_1e10_under_one_ulp(runs):
    d = rel(runs["ref_ulp"].rel_residual, runs["ref"].rel_residual)
    assert d[:12].max() <= 1e-12
    first = int(np.argmax(d > 1e-10))
    assert 16 <= first <= 28, first            # measured: 21
    assert d[:40].max() > 1e-3                   # fully decorrelated well before convergence


def test_contract_mode_within_1e10_inside_the_window(runs):
    d = rel(runs["rep"].rel_residual, runs["ref"].rel_residual)
    assert d[:17].max() <= 1e-10, d[:17].max()   # measured: 4.1e-12 at iteration 16


def test_contract_divergence_tracks_the_inherent_sensitivity(runs):
    d_rep = rel(runs["rep"].rel_residual, runs["ref"].rel_residual)
    d_ulp = rel(runs["ref_ulp"].rel_residual, runs["ref"].rel_residual)
    # compare growth: iteration at which each first exceeds 1e-10 and 1e-6
    for thr in (1e-10, 1e-6):
        i_rep = int(np.argmax(d_rep > thr))
        i_ulp = int(np.argmax(d_ulp > thr))
        assert abs(i_rep - i_ulp) <= 4, (thr, i_rep, i_ulp)


def test_both_modes_converge_with_counts_inside_the_sensitivity(runs, po):
    ref, rep, ulp = runs["ref"], runs["rep"], runs["ref_ulp"]
    assert ref.status == rep.status == ulp.status == "converged"
    assert abs(ref.n_iterations - ulp.n_iterations) <= 2
    assert abs(rep.n_iterations - ref.n_iterations) <= 2
    a, b, c1, c2 = runs["ops"]
    for sol in (ref, rep):
        tr = po.true_residual_factors(a, b, c1, c2, sol.V, sol.core, sol.W)
        assert tr <= 2e-8, tr
