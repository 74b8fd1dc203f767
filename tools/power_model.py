"""Power roofline of the assembly kernel on this pool's B200 (board limit 1 kW, `sw_power_cap`
under sustained C5 load).  Measures, each for ~4 s with nvidia-smi sampling:
  idle board power; the assembly's store pattern alone (store-only tile kernel); the C5
  per-entry arithmetic alone (register-only); and the real C5 assembly back to back,
then derives the energy per entry of each part and the power-bound rate
  entries/s <= (P_limit - P_idle) / (E_store + E_alu).

    python tools/power_model.py > profiles/r01_power_model.json
"""
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2602_10541_b200.build import build_microbench  # noqa: E402


def sample(fn, seconds=4.0):
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    t0 = time.time()
    clk.mark_begin()
    n = 0
    rates = []
    while time.time() - t0 < seconds:
        r = fn()
        if r is not None:
            rates.append(r)
        n += 1
    torch.cuda.synchronize()
    clk.mark_end()
    c = clk.stop()
    return c, (statistics.mean(rates) if rates else None), n


def main():
    out = {"gpu": torch.cuda.get_device_name(0)}
    try:
        q = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=power.limit", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=20).stdout.strip()
        out["power_limit_w"] = float(q)
    except Exception:
        out["power_limit_w"] = None
    torch.cuda.synchronize()
    c, _, _ = sample(lambda: time.sleep(0.05), 3.0)
    out["idle"] = c
    lib = C.CDLL(build_microbench())
    lib.mb_tile_store_bw.restype = C.c_int
    lib.mb_entry_rate.restype = C.c_int
    res = C.c_double()
    A = torch.empty(1 << 33, dtype=torch.float64, device="cuda")      # 64 GiB
    scratch = torch.zeros(4096, dtype=torch.float64, device="cuda")

    def store():
        lib.mb_tile_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(1 << 20), C.c_int64(1 << 20), 8192, 10,
                             C.byref(res))
        return res.value * 1e9                                           # B/s
    c, rate, _ = sample(store)
    out["store"] = {"bytes_per_s": rate, "clocks": c}

    def alu():
        lib.mb_entry_rate(C.c_void_p(scratch.data_ptr()), 400_000, C.byref(res))
        return res.value                                                 # entries/s
    c, rate, _ = sample(alu)
    out["c5_alu"] = {"entries_per_s": rate, "clocks": c}
    del A
    torch.cuda.empty_cache()

    # the real thing: C5 assembly (fls_features_assemble) back to back
    import workloads as wl
    from paper_2602_10541_b200 import fls
    p = wl.make_problem("c5_biharm3d", "full")
    F, R, d = p.n_features, p.n_rows, p.dim
    blocks = [fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight, torch.from_numpy(b.values).cuda(),
                        torch.from_numpy(b.fields).cuda() if b.fields is not None else None) for b in p.blocks]
    ctx = fls.Context()
    bset = fls.BlockSet(blocks, d)
    lda = fls.round_up(R, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")

    def asm():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        e1.record(ctx.stream)
        e1.synchronize()
        return R * F / (e0.elapsed_time(e1) / 1e3)
    for _ in range(3):
        asm()
    c, rate, n = sample(asm)
    out["c5_assembly"] = {"entries_per_s": rate, "steps": n, "clocks": c}

    idle = out["idle"]["power_w_median"]
    e_store = (out["store"]["clocks"]["power_w_median"] - idle) / out["store"]["bytes_per_s"] * 8.0
    e_alu = (out["c5_alu"]["clocks"]["power_w_median"] - idle) / out["c5_alu"]["entries_per_s"]
    lim = out["power_limit_w"] or 1000.0
    bound = (lim - idle) / (e_store + e_alu)
    out["model"] = {"idle_w": idle, "store_nj_per_entry": e_store * 1e9, "alu_nj_per_entry": e_alu * 1e9,
                    "power_limit_w": lim, "power_bound_entries_per_s": bound,
                    "c5_assembly_frac_of_power_bound": rate / bound,
                    "c5_assembly_power_predicted_w": idle + rate * (e_store + e_alu),
                    "note": "store/ALU probes run alone at full clock; the real kernel runs both "
                            "at once under sw_power_cap"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
