"""Golden residual histories of the CPU oracle at the BASELINE configs C2-C5.

TEST INFRASTRUCTURE. Runs the oracle (oracle/sk_oracle.c, OpenMP build
libsk_oracle_mt.so: bitwise the serial build) once per config and arithmetic mode
and writes tests/golden/config<N>_<mode>.json:

    {"config", "mode", "status", "iterations", "rel_residual" (17-digit floats),
     "max_iter", "window" (null for a full run), "paths", "core_fro", "oracle_s",
     "host": {"cpu", "nproc", "threads"}}

REPRODUCIBLE is the contract the GPU executes bit for bit; REFERENCE_ORDER follows
the reference loop by loop (factorized_solvers.cpp:134-192, :268-381). The GPU tests
(tests/test_gpu_configs.py) compare against these files, so the box never needs to
rerun the oracle. Lanczos configs (C3, C5) run "lean" (only the last basis blocks are
kept: history and core only), which is what lets C5 (108 GB of bases) run in host RAM.
C4's bases (~60 GB per mode) exceed this container, so its goldens cover the leading
window of iterations (--window).

Usage (repo root):  python tests/golden/make_config_golden.py 3 5 4 2 [--threads N]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))

WINDOWS = {4: 30}  # config -> leading iterations when the full run does not fit this host


def host_info(threads):
    cpu = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count(), "threads": threads}


def oracle_inputs(idx):
    """The BASELINE config's inputs from the oracle's own generators (bitwise the
    product's: tests/test_library.py::test_generators_match_oracle)."""
    import numpy as np
    from oracle import pyoracle as po
    seed = 1234
    if idx == 1:
        a = po.laplacian_2d(64)
        c1 = po.random_rhs(4096, 1, seed)
        c1 /= np.linalg.norm(c1)
        c2 = po.random_rhs(4096, 1, seed + 1)
        c2 /= np.linalg.norm(c2)
        return po.CG, a, a, c1, c2, 500
    if idx == 2:
        a = po.convection_diffusion_2d(256, (10.0, 10.0))
        b = po.convection_diffusion_2d(256, (10.0, -10.0))
        return po.BICGSTAB, a, b, po.random_rhs(65536, 4, seed), po.random_rhs(65536, 4, seed + 1), 0
    if idx == 3:
        a = po.laplacian_2d(1024)
        return po.CG_LYAPUNOV, a, None, po.random_rhs(1 << 20, 1, seed), None, 0
    if idx == 4:
        a = po.convection_diffusion_3d(128, (5.0, 2.5, 1.25))
        b = po.convection_diffusion_3d(64, (0.0, 0.0, 0.0))
        return po.BICGSTAB, a, b, po.random_rhs(128 ** 3, 8, seed), po.random_rhs(64 ** 3, 8, seed + 1), 0
    if idx == 5:
        a = po.laplacian_2d(4096)
        return po.CG, a, a, po.random_rhs(1 << 24, 2, seed), po.random_rhs(1 << 24, 2, seed + 1), 200
    raise ValueError(idx)


def run(idx, mode_name, threads, window=None, perturb=False):
    import numpy as np
    from oracle import pyoracle as po
    po.use_threads(threads)
    method, a, b, c1, c2, max_iter = oracle_inputs(idx)
    if perturb == "all":  # every entry of C1 scaled by (1 + 2^-52): rounding-level change everywhere
        c1 = c1 * (1.0 + 2.0 ** -52)
    elif perturb:  # one entry of C1 moved by one ulp: the run's own sensitivity
        c1 = c1.copy()
        c1[5, 0] = np.nextafter(c1[5, 0], np.inf)
    if window:
        max_iter = window
    mode = po.REPRODUCIBLE if mode_name == "reproducible" else po.REFERENCE_ORDER
    lean = method != po.BICGSTAB
    t0 = time.time()
    sol = po.solve(method, a, b, c1, c2, po.Config(eps_tol=1e-8, max_iter=max_iter), mode, lean=lean)
    dt = time.time() - t0
    out = {"config": f"C{idx}", "mode": mode_name, "status": sol.status,
           "iterations": int(sol.n_iterations), "max_iter": int(max_iter), "window": window,
           "rel_residual": [float(x) for x in sol.rel_residual], "paths": sol.paths,
           "core_shape": list(sol.core.shape), "core_fro": float(np.linalg.norm(sol.core)),
           "oracle_s": dt, "host": host_info(threads)}
    path = os.path.join(HERE, f"config{idx}_{mode_name}{('_ulpall' if perturb == 'all' else '_ulp') if perturb else ''}.json")
    out["perturbed"] = bool(perturb)
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"C{idx} {mode_name}: {sol.status} after {sol.n_iterations} iterations, "
          f"rel {sol.rel_residual[-1]:.6e}, {dt:.1f} s -> {path}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", type=int)
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--modes", default="reproducible,reference_order")
    ap.add_argument("--window", type=int, default=None, help="override the leading-iteration window")
    ap.add_argument("--perturb", action="store_true", help="move C1[5,0] by one ulp (sensitivity run; file suffix _ulp)")
    ap.add_argument("--perturb-all", action="store_true", help="scale all of C1 by 1 + 2^-52 (file suffix _ulpall)")
    ap.add_argument("--full", action="store_true", help="no window (config 4 needs ~60 GB of host memory per mode)")
    ap.add_argument("--out-dir", default=None, help="write the JSON files here instead of tests/golden")
    args = ap.parse_args()
    if args.out_dir:
        HERE = args.out_dir
        os.makedirs(HERE, exist_ok=True)
    for idx in args.configs:
        for mode_name in args.modes.split(","):
            run(idx, mode_name, args.threads, None if args.full else (args.window or WINDOWS.get(idx)), 'all' if args.perturb_all else args.perturb)
