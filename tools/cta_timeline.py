"""Per-CTA timeline of the assembly kernel in a steady-state step (diagnostic build).

Needs the FLS_DIAG_CTATIME=1 variant (each CTA's thread 0 records %globaltimer at entry, after
its griddepcontrol.wait, after the first chunk's records, at the end, plus its SM and row block):

    python -m paper_2602_10541_b200.build --variant ctatime -D FLS_DIAG_CTATIME=1
    FLS_LIB=$PWD/paper_2602_10541_b200/libfls_ctatime.so python tools/cta_timeline.py c2_poisson2d

Replays a graph of 10 fls_features_assemble calls (the bench's call) and reads the last call's
records.  Prints one JSON line per config: the kernel window, per row block the median phases
(wait, records, body), the spread of CTA start / end times, and how many SM slots are busy
over the window (deciles).
"""
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import _abi, fls  # noqa: E402

SLOTS = 8


def main(names):
    lib = _abi.load()
    rd = lib.fls_diag_cta
    rd.restype = C.c_int
    rd.argtypes = [C.c_void_p, C.c_longlong]
    s = torch.cuda.Stream()
    for name in names:
        p = wl.make_problem(name, "full")
        F, R, d = p.n_features, p.n_rows, p.dim
        ctx = fls.Context(stream=s)
        bset = fls.BlockSet([fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight,
                                       torch.from_numpy(b.values).cuda(),
                                       torch.from_numpy(b.fields).cuda() if b.fields is not None else None)
                             for b in p.blocks], d)
        lda = fls.round_up(R, 4)
        Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
        W = torch.empty((F, d), dtype=torch.float64, device="cuda")
        b = torch.empty((F,), dtype=torch.float64, device="cuda")
        fn = lambda: fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    fn()
            buf = np.zeros(SLOTS * 65536, dtype=np.uint64)
            res = []
            for rep in range(5):
                for _ in range(20):
                    g.replay()
                torch.cuda.synchronize()
                assert rd(buf.ctypes.data, buf.nbytes) == 0
                res.append(buf.reshape(-1, SLOTS).copy())
        if os.environ.get("CTA_DUMP"):
            np.save(os.path.join(os.environ["CTA_DUMP"], f"cta_{name}.npy"), res[-1])
        out = {"config": name}
        phases = {}
        for r in res:
            n = int(np.count_nonzero(r[:, 3]))
            r = r[:n].astype(np.int64)
            t0 = r[:, 0].min()
            t = r[:, :4] - t0
            phases.setdefault("window_us", []).append(t[:, 3].max() / 1e3)
            for q in sorted(set(r[:, 5].tolist())):
                m = r[:, 5] == q
                tq = t[m]
                key = f"block{q}"
                phases.setdefault(key + "_ctas", []).append(int(m.sum()))
                phases.setdefault(key + "_wait_us", []).append(float(np.median(tq[:, 1] - tq[:, 0])) / 1e3)
                t6 = r[m, 6].astype(np.int64) - t0
                phases.setdefault(key + "_points_us", []).append(float(np.median(t6 - tq[:, 0])) / 1e3)
                phases.setdefault(key + "_records_us", []).append(float(np.median(tq[:, 2] - tq[:, 1])) / 1e3)
                phases.setdefault(key + "_body_us", []).append(float(np.median(tq[:, 3] - tq[:, 2])) / 1e3)
                phases.setdefault(key + "_start_p0_p50_p100_us", []).append(
                    [float(np.percentile(tq[:, 0], v)) / 1e3 for v in (0, 50, 100)])
                phases.setdefault(key + "_end_p0_p50_p100_us", []).append(
                    [float(np.percentile(tq[:, 3], v)) / 1e3 for v in (0, 50, 100)])
            # busy CTA slots over the window (deciles)
            W_ = t[:, 3].max()
            busy = []
            for k in range(10):
                tm = W_ * (k + 0.5) / 10
                busy.append(int(((t[:, 0] <= tm) & (t[:, 3] > tm)).sum()))
            phases.setdefault("busy_ctas_by_decile", []).append(busy)
            sm = r[:, 4]
            phases.setdefault("ctas_per_sm_min_max", []).append(
                [int(np.bincount(sm).min()), int(np.bincount(sm).max())])
        for k, v in phases.items():
            if isinstance(v[0], list):
                out[k] = v[len(v) // 2]
            else:
                out[k] = round(statistics.median(v), 3)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2_poisson2d"])
