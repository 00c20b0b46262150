"""On-disk formats: the native Matrix Market writers are pinned
byte-for-byte against the reference's own matrix_market.cpp (built by
oracle/build_ref.sh into oracle/_ref/, CPU), the Python reader against the
reference's reader; on the GPU, the factor files streamed from HBM equal the
copied factors and the history CSV follows write_history_csv (bench.cpp:179-193)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2605_28274_b200 as sk
from oracle import pyoracle as po

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libsylkrylov_ref.so")
i64p, f64p = C.POINTER(C.c_int64), C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF) and os.path.isdir("/root/reference/proj/src"):
        os.system(os.path.join(os.path.dirname(REF), "..", "build_ref.sh") + " > /dev/null")
    if not os.path.exists(REF):
        pytest.skip("reference library not built (no /root/reference here)")
    lib = C.CDLL(REF)
    if not hasattr(lib, "ref_write_mm_csr"):
        pytest.skip("reference library predates the Matrix Market entry points")
    lib.ref_read_mm_csr.restype = C.c_int64
    return lib


def P(a, t=f64p):
    return a.ctypes.data_as(t)


def csr(a):
    return sk.SparseMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values)


def odd_values(n, seed):
    """Values that stress %.17g: signed zeros, subnormals, huge and tiny magnitudes."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    v[::7] = -0.0
    v[1::11] = 5e-324
    v[2::13] = 1.0 / 3.0
    return v


@pytest.mark.parametrize("g", [2, 3, 17])
def test_csr_writer_matches_reference(ref, tmp_path, g):
    a = po.laplacian_2d(g)
    a = po.Csr(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, odd_values(a.values.size, g))
    ours, theirs = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    sk.write_matrix_market(csr(a), ours)
    assert ref.ref_write_mm_csr(C.c_int64(a.n_rows), C.c_int64(a.n_cols), C.c_int64(a.values.size),
                                P(a.row_ptr, i64p), P(a.col_idx, i64p), P(a.values), theirs.encode()) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()


@pytest.mark.parametrize("shape", [(0, 0), (1, 1), (5, 3), (300, 7)])
def test_dense_writer_matches_reference(ref, tmp_path, shape):
    x = odd_values(shape[0] * shape[1], 7).reshape(shape, order="F")
    ours, theirs = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    sk.write_matrix_market(x, ours)
    xf = np.asfortranarray(x)
    assert ref.ref_write_mm_dense(C.c_int64(shape[0]), C.c_int64(shape[1]), P(xf), theirs.encode()) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_dense_writer_parallel_chunks_in_order(tmp_path):
    # large enough for the multi-thread formatter; the file must still be in column-major order
    x = np.arange(600_000, dtype=np.float64).reshape((200_000, 3), order="F") * 0.5
    p = str(tmp_path / "x.mtx")
    sk.write_matrix_market(x, p)
    assert np.array_equal(sk.read_matrix_market(p), x)


@pytest.mark.parametrize("sym", ["general", "symmetric"])
def test_reader_matches_reference(ref, tmp_path, sym):
    rng = np.random.default_rng(3)
    n = 40
    ent = {}
    for _ in range(150):
        i, j = sorted(rng.integers(0, n, 2).tolist(), reverse=True) if sym == "symmetric" else \
            rng.integers(0, n, 2).tolist()
        ent[(i, j)] = float(rng.standard_normal())
    p = str(tmp_path / "m.mtx")
    with open(p, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real {sym}\n% comment\n\n{n} {n} {len(ent)}\n")
        for (i, j), v in ent.items():
            f.write(f"{i + 1} {j + 1} {v!r}\n")
    ours = sk.read_matrix_market(p)
    dims = np.zeros(3, dtype=np.int64)
    assert ref.ref_read_mm_csr(p.encode(), P(dims, i64p), None, None, None) >= 0
    rp = np.zeros(dims[0] + 1, dtype=np.int64)
    ci = np.zeros(dims[2], dtype=np.int64)
    v = np.zeros(dims[2])
    ref.ref_read_mm_csr(p.encode(), P(dims, i64p), P(rp, i64p), P(ci, i64p), P(v))
    assert (ours.n_rows, ours.n_cols) == (dims[0], dims[1])
    assert np.array_equal(ours.row_ptr, rp) and np.array_equal(ours.col_idx, ci)
    assert np.array_equal(ours.values, v)


def test_reader_rejects_malformed(tmp_path):
    p = str(tmp_path / "bad.mtx")
    for text in ["%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n",
                 "%%MatrixMarket matrix array real symmetric\n1 1\n1\n",
                 "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
                 "not a header\n"]:
        with open(p, "w") as f:
            f.write(text)
        with pytest.raises(sk.ParseError):
            sk.read_matrix_market(p)


def test_writer_io_error():
    with pytest.raises(sk.IoError):
        sk.write_matrix_market(np.zeros((2, 2)), "/nonexistent-dir/x.mtx")


@pytest.mark.gpu
@pytest.mark.parametrize("s", [1, 2])
def test_factor_files_and_history(tmp_path, s):
    a = po.laplacian_2d(24)
    c1, c2 = po.random_rhs(a.n_rows, s, 11), po.random_rhs(a.n_rows, s, 12)
    A = csr(a)
    cfg = sk.SolverConfig(eps_tol=1e-8)
    sol = sk.factorized_cg(A, A, c1, c2, cfg)
    V, core, W = sol.V, sol.core, sol.W
    # Matrix Market triple: identical bytes to the in-memory writer of the copied factors
    d = tmp_path / "mtx"
    sol.write_factors(str(d), "mtx")
    for name, m in [("V", V), ("core", core), ("W", W)]:
        sk.write_matrix_market(m, str(tmp_path / f"{name}_direct.mtx"))
        assert open(d / f"{name}.mtx", "rb").read() == open(tmp_path / f"{name}_direct.mtx", "rb").read()
        assert np.array_equal(sk.read_matrix_market(str(d / f"{name}.mtx")), m)
    # binary sidecar round trip
    b = tmp_path / "bin"
    sol.write_factors(str(b), "binary")
    for name, m in [("V", V), ("core", core), ("W", W)]:
        assert np.array_equal(sk.read_factor(str(b / f"{name}.skb")), m)
    # column-range copies agree with the whole-basis copy
    buf = np.zeros((sol.n, 3), order="F")
    sk.lib().sk_solution_copy_V_cols(sol._h, C.c_int64(1), C.c_int64(3), buf.ctypes.data_as(f64p))
    assert np.array_equal(buf, V[:, 1:4])
    # history.csv: header + one row per record, cumulative time = running sum
    p = str(tmp_path / "history.csv")
    sol.write_history_csv(p)
    lines = open(p).read().splitlines()
    assert lines[0] == "iteration,rel_residual,cumulative_time_s,basic_s,krylov_s,trunc_s"
    recs = sol.history.records
    assert len(lines) == 1 + len(recs)
    for ln, r in zip(lines[1:], recs):
        f = ln.split(",")
        assert int(f[0]) == r.iteration and float(f[1]) == r.rel_residual
    # meta.json of the CLI (main.cpp:146-239)
    meta = sk.write_solution(str(tmp_path / "out"), "f-cg", sol, A, A, c1, c2, cfg, seed=11)
    on_disk = json.load(open(tmp_path / "out" / "meta.json"))
    assert on_disk == json.loads(json.dumps(meta))
    assert meta["status"] == "converged" and meta["final_true_residual"] < 1e-7
    assert meta["ranks"] == {"rank": min(sol.rv, sol.rw), "v_cols": sol.rv, "w_cols": sol.rw}
    sol.free()
