"""Measure the roofline denominators of the assembly path on the GPU box:
store-only HBM bandwidth (assembly store pattern), DFMA/s, and the register-only rate of the
C5 kernel's per-entry arithmetic, each with nvidia-smi clocks sampled while it runs.

    python tools/roofline_probe.py > profiles/roofline_probe_r01.json
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2602_10541_b200.build import build_microbench  # noqa: E402


def main():
    lib = C.CDLL(build_microbench())
    for f in (lib.mb_store_bw, lib.mb_dfma_rate, lib.mb_entry_rate, lib.mb_tile_store_bw,
              lib.mb_chunk_store_bw):
        f.restype = C.c_int
    out = {"gpu": torch.cuda.get_device_name(0)}
    scratch = torch.zeros(4096, dtype=torch.float64, device="cuda")
    n = 8 * (1 << 30)                                   # 64 GiB of fp64
    A = torch.empty(n, dtype=torch.float64, device="cuda")
    res = C.c_double()
    for name, call in [
        ("store_gbs", lambda: lib.mb_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(n), 20, C.byref(res))),
        ("tile_store_gbs", lambda: lib.mb_tile_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(1 << 20),
                                                         C.c_int64(1 << 20), 8192, 10, C.byref(res))),
        ("chunk_store_gbs", lambda: lib.mb_chunk_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(n), 20,
                                                          C.byref(res))),
        ("dfma_per_s", lambda: lib.mb_dfma_rate(C.c_void_p(scratch.data_ptr()), 2_000_000, C.byref(res))),
        ("c5_entry_alu_per_s", lambda: lib.mb_entry_rate(C.c_void_p(scratch.data_ptr()), 400_000, C.byref(res))),
    ]:
        clk = ClockSampler(0)
        clk.start()
        st = call()
        torch.cuda.synchronize()
        out[name] = res.value
        out[name + "_clocks"] = clk.stop()
        out[name + "_status"] = st
    lib.mb_op_rate.restype = C.c_int
    for op, name in enumerate(["dadd", "dmul", "dfma", "frnd_dadd", "f2i_i2f", "c5_entry_frnd"]):
        st = lib.mb_op_rate(op, C.c_void_p(scratch.data_ptr()), 200_000 if op < 5 else 400_000,
                            C.byref(res))
        torch.cuda.synchronize()
        out[f"op_{name}_per_s"] = res.value
    lib.mb_dmma_rate.restype = C.c_int
    r2 = C.c_double()
    for mode, name in enumerate(["dmma_only", "dmma_plus_dfma", "dfma_only"]):
        st = lib.mb_dmma_rate(mode, C.c_void_p(scratch.data_ptr()), 200_000, C.byref(res), C.byref(r2))
        torch.cuda.synchronize()
        # one m8n8k4 DMMA = 8*8*4 = 256 FMAs
        out[f"{name}_dmma_fma_per_s"] = res.value * 256
        out[f"{name}_dfma_per_s"] = r2.value
        out[f"{name}_status"] = st
    # power split: each probe run back to back for ~4 s with clocks / power sampled
    if os.environ.get("FLS_POWER_PROBE", "1") == "1":
        import time as _t
        for name, call in [
            ("power_store", lambda: lib.mb_tile_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(1 << 20),
                                                         C.c_int64(1 << 20), 8192, 10, C.byref(res))),
            ("power_chunk_store", lambda: lib.mb_chunk_store_bw(C.c_void_p(A.data_ptr()), C.c_int64(n), 20,
                                                                C.byref(res))),
            ("power_dmma", lambda: lib.mb_dmma_rate(0, C.c_void_p(scratch.data_ptr()), 1_000_000,
                                                    C.byref(res), C.byref(r2))),
            ("power_dfma", lambda: lib.mb_dmma_rate(2, C.c_void_p(scratch.data_ptr()), 1_000_000,
                                                    C.byref(res), C.byref(r2))),
            ("power_alu", lambda: lib.mb_entry_rate(C.c_void_p(scratch.data_ptr()), 400_000, C.byref(res))),
        ]:
            clk = ClockSampler(0)
            clk.start()
            t0 = _t.time()
            rates, rates2 = [], []
            while _t.time() - t0 < 4.0:
                call()
                torch.cuda.synchronize()
                rates.append(res.value)
                rates2.append(r2.value)
            out[name] = {"rate": sum(rates) / len(rates), "rate2": sum(rates2) / len(rates2),
                         "clocks": clk.stop()}
    mhz = out["dfma_per_s_clocks"]["sm_mhz"]
    if mhz:
        out["dfma_per_clk_per_sm"] = out["dfma_per_s"] / (mhz * 1e6) / torch.cuda.get_device_properties(0).multi_processor_count
    out["c5_entry_alu_gbs_equiv"] = out["c5_entry_alu_per_s"] * 8 / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
