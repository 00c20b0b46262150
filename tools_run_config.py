"""Run one BASELINE config on the GPU and print a JSON summary (time-to-tolerance)."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2605_28274_b200 as sk
from paper_2605_28274_b200.problems import baseline_config

idx = int(sys.argv[1])
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = baseline_config(idx)
scfg = sk.SolverConfig(eps_tol=cfg.eps_tol, max_iter=max_iter if max_iter is not None else cfg.max_iter)
prob = sk.ResidentProblem(cfg.method, cfg.a, cfg.b, cfg.c1, cfg.c2, gpu=sk.GpuOptions(profile=True))
out = {}
for rep in range(2):
    t0 = time.perf_counter()
    sol = prob.solve(scfg)
    wall = time.perf_counter() - t0
    out = {"config": cfg.name, "status": sol.status, "iterations": sol.history.iterations(),
           "final_rel": sol.history.final_rel_residual(), "device_s": sol.stats["device_time_s"], "wall_s": wall,
           "rv": sol.rv, "rw": sol.rw, "paths": sol.stats["paths"],
           "classes": {k: v for k, v in sol.stats["classes"].items() if v["launches"]}}
    hist = sol.history.rel_residuals()
    sol.free()
print(json.dumps(out))
json.dump({"config": cfg.name, "rel_residual": hist.tolist()}, open(f"gpurun_out/hist_{cfg.name}.json", "w"))
