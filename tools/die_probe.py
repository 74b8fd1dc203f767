"""Does the die a store lands on change its energy?  (tools/die_probe.cu; tuning evidence only)

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
         -o tools/_die_probe.so tools/die_probe.cu
    python tools/die_probe.py [GB]

Prints one JSON line: the SM -> die split, the near / far L2-hit latencies, the chunk
classification's repeatability, and for each write mode (mixed, own die, other die) the write
bandwidth, the board power and the energy per byte above idle.
"""
import ctypes
import json
import os
import sys
import threading
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "_die_probe.so"))
P = ctypes.c_void_p


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def check(rc):
    if rc != 0:
        raise RuntimeError(f"cuda error {rc}")


class Power:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.samples = []
        self.run = False

    def _loop(self):
        while self.run:
            self.samples.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            time.sleep(0.01)

    def __enter__(self):
        self.samples, self.clk, self.run = [], [], True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.run = False
        self.t.join()


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    dev = torch.device("cuda", 0)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    nchunk = int(gb * 2**30) // 2048
    buf = torch.zeros(nchunk * 256, dtype=torch.int64, device=dev)

    # 1. SM -> die from a 256-chunk sample seen by every SM
    ns, grid = 256, nsm * 4
    lat = torch.zeros(grid * ns, dtype=torch.float32, device=dev)
    smc = torch.zeros(grid, dtype=torch.int32, device=dev)
    check(lib.die_lat(ptr(buf), ns, 32, ptr(lat), ptr(smc), grid))
    torch.cuda.synchronize()
    L = lat.view(grid, ns).cpu().numpy()
    sm_ids = smc.cpu().numpy()
    per_sm = {}
    for c, s in enumerate(sm_ids):
        per_sm.setdefault(int(s), []).append(L[c])
    sms = sorted(per_sm)
    M = np.stack([np.mean(per_sm[s], axis=0) for s in sms])       # (SMs, chunks)
    near = M < np.median(M, axis=0, keepdims=True)                # near pattern per SM
    ref = near[0]
    same = (near == ref[None, :]).mean(axis=1) > 0.5
    die_of_sm = np.zeros(max(sms) + 1, dtype=np.int32)
    for s, sd in zip(sms, same):
        die_of_sm[s] = 0 if sd else 1
    lat_near = float(np.median(M[near]))
    lat_far = float(np.median(M[~near]))
    thr = 0.5 * (lat_near + lat_far)

    # 2. every chunk, from whichever SM takes it
    def classify():
        la = torch.zeros(nchunk, dtype=torch.float32, device=dev)
        sm = torch.zeros(nchunk, dtype=torch.int32, device=dev)
        check(lib.die_classify(ptr(buf), ctypes.c_longlong(nchunk), 8, ptr(la), ptr(sm), nsm * 4))
        torch.cuda.synchronize()
        la, sm = la.cpu().numpy(), sm.cpu().numpy()
        d = die_of_sm[sm]
        return np.where(la < thr, d, 1 - d), la

    t0 = time.time()
    dA, la = classify()
    dB, _ = classify()
    t_cls = time.time() - t0
    agree = float((dA == dB).mean())
    dies = dA
    lists = np.concatenate([np.nonzero(dies == 0)[0], np.nonzero(dies == 1)[0]]).astype(np.int64)
    n0 = int((dies == 0).sum())
    n1 = nchunk - n0
    lists_d = torch.from_numpy(lists).to(dev)
    dmap = torch.from_numpy(die_of_sm).to(dev)
    ctr = torch.zeros(3, dtype=torch.int64, device=dev)

    # 3. writes: idle power, then each mode ~3 s, two rounds
    pw = Power()
    time.sleep(1.0)
    with pw as p:
        time.sleep(1.5)
    idle = float(np.median(p.samples))

    def run(mode, passes):
        ctr.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib.die_write(ptr(buf), ptr(lists_d), ctypes.c_longlong(n0), ctypes.c_longlong(n1),
                            ptr(dmap), mode, passes, ptr(ctr), nsm * 8, 256))
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    t1 = run(0, 2)
    passes = max(2, int(3.0 / (t1 / 2)))
    out = {"n_sm": nsm, "sm_die0": int((die_of_sm[sms] == 0).sum()), "sm_die1": int((die_of_sm[sms] == 1).sum()),
           "lat_near_cyc": lat_near, "lat_far_cyc": lat_far, "chunks": nchunk, "chunks_die0": n0,
           "classify_repeat_agreement": agree, "classify_s": t_cls, "idle_w": idle, "modes": []}
    names = {0: "mixed", 1: "own die", 2: "other die"}
    for rnd in range(2):
        for mode in (0, 1, 2):
            run(mode, 2)
            with pw as p:
                t = run(mode, passes)
            nbytes = 2048.0 * (n0 + n1) * passes   # modes 1/2 write each die's list `passes` times too
            w = float(np.mean(p.samples))   # energy = mean power x time (a die may finish first)
            out["modes"].append({"mode": names[mode], "round": rnd, "s": t, "gbs": nbytes / t / 1e9,
                                 "power_w": w, "sm_mhz": float(np.median(p.clk)),
                                 "pj_per_byte_above_idle": (w - idle) / (nbytes / t) * 1e12})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
