"""Offline oracle artifacts for full-size solve parity: for each BASELINE config
the CPU oracle assembles [A | b] at full size (C5: its 262,144-row solve subset), solves with
unblocked Householder QR (C5 with the tau = 1e-10 relative ridge, reading A16) and evaluates u
at the config's 10,000 held-out points.  Calls only oracle/ and workloads/ -- no value comes
from the CUDA path.  Output: tests/golden/oracle_u_<config>.npz (u_test, timings, host info).

    python tools/make_oracle_artifacts.py c3_poisson5d c4_heat2d c5_biharm3d
"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as wl  # noqa: E402

SOLVE_ROWS = {"c5_biharm3d": 262_144}


def main(names):
    for name in names:
        kw = {"n_int": SOLVE_ROWS[name]} if name in SOLVE_ROWS else {}
        p = wl.make_problem(name, "full", **kw)
        W, b = p.parity_features()
        t0 = time.time()
        A, r, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
        t1 = time.time()
        beta, res, rd = oracle.lstsq(A, r, ridge_rel=p.ridge_rel)
        t2 = time.time()
        del A
        Xt = p.test_points(10_000)
        u = oracle.evaluate(W, b, beta, Xt)
        t3 = time.time()
        meta = {"config": name, "rows": p.n_rows, "features": p.n_features,
                "ridge_rel": p.ridge_rel, "resid": res, "assemble_s": t1 - t0, "lstsq_s": t2 - t1,
                "eval_s": t3 - t2, "threads": oracle.max_threads(), "host": platform.node(),
                "cpu": platform.processor(), "script": "tools/make_oracle_artifacts.py"}
        out = os.path.join(ROOT, "tests", "golden", f"oracle_u_{name}.npz")
        np.savez_compressed(out, u_test=u, meta=json.dumps(meta))
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3_poisson5d", "c4_heat2d"])
