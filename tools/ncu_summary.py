"""Summarise ncu outputs into profiles/ (tracked): the per-launch list (share of the step per
kernel) and the key metrics of one `--set full` capture of the top kernel.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.md
    python tools/ncu_summary.py full gpurun_out/prof_c5.ncu-rep --algo-bytes N > profiles/r01_assemble_ncu.md
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_write.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    by = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r["Metric Unit"]]
        by.setdefault(r["Kernel Name"], []).append(v * scale)
    tot = sum(sum(v) for v in by.values())
    print("| kernel | launches | mean ms | total ms | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.4f} | {sum(v):.3f} | {100 * sum(v) / tot:.2f}% |")
    print(f"\n(cold-cache, serialised ncu replay; compare shares, not absolutes) total {tot:.3f} ms")


def full(path, algo_bytes):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        res[name] = d
    for name, d in res.items():
        print(f"### `{name}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k, (v, u) in d.items():
            print(f"| {k} | {v} | {u} |")
        if algo_bytes:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * _mult(d["dram__bytes_read.sum"][1])
            wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * _mult(d["dram__bytes_write.sum"][1])
            print(f"\ntraffic (read + write) = {rd + wr:.4e} B per launch; algorithmic = {algo_bytes:.4e} B "
                  f"(ratio {(rd + wr) / algo_bytes:.4f})")
            print("\n```json\n" + json.dumps({"traffic_bytes": rd + wr, "algo_bytes": algo_bytes}) + "\n```")
        print()


def _mult(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--algo-bytes", type=float, default=None)
    a = ap.parse_args()
    launches(a.path) if a.mode == "launches" else full(a.path, a.algo_bytes)
