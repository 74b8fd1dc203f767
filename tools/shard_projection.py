"""Per-shard assembly rate of the C5 scaling sweep, measured on ONE GPU (a projection, not a
multi-GPU measurement).

Row-sharded assembly has no collective: at P GPUs rank r assembles its own
contiguous 2,097,152 / P rows into its own HBM, under its own 1 kW board limit.  This script
times exactly that per-rank workload on one B200 (`bench.py --rows R/P`, the same fused call and
launch plan a rank runs) for P = 1, 2, 4, 8, and reports per P: the per-GPU entries/s, the
fraction of the copy peak, and the aggregate P x per-GPU rate that the driver's scaling run would
see if the GPUs do not interact.  It is labelled a projection everywhere it is quoted; the
scaling run itself (`bench.py --gpus P` under torchrun) is the measurement.

    python tools/shard_projection.py [--steps 20] [--sustained-s 0] > profiles/<round>_shard_projection.jsonl
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = 2_097_152


def run(rows, steps, warmup):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--rows", str(rows), "--steps", str(steps),
           "--warmup", str(warmup), "--no-e2e", "--no-solve", "--no-per-config", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--sustained-s", type=float, default=0.0,
                    help="also time about this many seconds of steps back to back (power-capped regime)")
    a = ap.parse_args()
    base = {}
    for P in (1, 2, 4, 8):
        rows = ROWS // P
        legs = {"short": run(rows, a.steps, 3)}
        if a.sustained_s > 0:
            n = max(a.steps, int(a.sustained_s * 1e3 / legs["short"]["ms_per_step"]))
            legs["sustained"] = run(rows, n, 3)
        rec = {"P": P, "rows_per_gpu": rows, "kind": "projection from one GPU (per-rank workload)"}
        for k, d in legs.items():
            per_gpu = d["value"]
            base.setdefault(k, per_gpu)
            rec[k] = {"steps": d["steps"], "ms_per_step": d["ms_per_step"],
                      "entries_per_s_per_gpu": per_gpu, "frac_of_copy_peak": d["roofline"]["frac"],
                      "projected_aggregate_entries_per_s": P * per_gpu,
                      "projected_efficiency_vs_P1": per_gpu / base[k],
                      "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"]}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
