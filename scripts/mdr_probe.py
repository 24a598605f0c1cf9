"""MDR (row f2) throughput on the GPU: refactor of a 257^3 f64 multisine field (32 planes), then a full
retrieval (request at 1e-6 of the range, INF) and reconstruction — wall time of the public calls
(host segments, as the reference's store), median of 3; the reference library's refactor and
reconstruction on a 65^3 sample for scale (oracle/_ref, host cores)."""
import json, os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import paper_2401_05994_b200 as mg
from paper_2401_05994_b200 import mdr


def field(n):
    from oracle import binding
    return binding.get("restatement").multisine((n, n, n)) if hasattr(binding, "get") else None


def run(u, reps=3):
    ts_r, ts_c = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        store = mdr.refactor(u, planes=32)
        t1 = time.perf_counter()
        m = store.manifest
        st = mdr.make_initial_state(m)
        rng = float(u.max() - u.min())
        req = mdr.request(m, 1e-6 * rng, mg.Norm.inf, 0.0, st)
        t2 = time.perf_counter()
        got = mdr.reconstruct(m, lambda l, p: store.segments[l][p], req, st, mg.Norm.inf, 0.0)
        t3 = time.perf_counter()
        ts_r.append(t1 - t0)
        ts_c.append(t3 - t2)
        err = float(np.max(np.abs(got - u)))
    return sorted(ts_r)[reps // 2], sorted(ts_c)[reps // 2], err, req.total_bytes


n = int(sys.argv[1]) if len(sys.argv) > 1 else 257
x = np.linspace(0, 1, n)
X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
u = np.sin(6.1 * X) * np.cos(4.3 * Y) + 0.5 * np.sin(9.7 * Z + X) + 0.1 * X * Y
tr, tc, err, nbytes = run(u)
res = {"shape": [n] * 3, "refactor_s": round(tr, 4), "refactor_gbs": round(u.nbytes / tr / 1e9, 2),
       "reconstruct_s": round(tc, 4), "reconstruct_gbs": round(u.nbytes / tc / 1e9, 2),
       "retrieved_bytes": int(nbytes), "max_err_over_range": err / float(u.max() - u.min())}
try:
    from oracle import binding
    if binding.available("reference"):
        v = u[:65, :65, :65].copy() if n >= 65 else u
        t0 = time.perf_counter()
        ref = binding.mdr_refactor(np.ascontiguousarray(v), 32)
        res["reference_refactor_65cubed_s"] = round(time.perf_counter() - t0, 4)
        res["reference_refactor_65cubed_gbs"] = round(v.nbytes / (time.perf_counter() - t0) / 1e9, 4)
except Exception as e:  # pragma: no cover
    res["reference"] = f"unavailable: {e}"
print(json.dumps(res))
