"""CPU stand-in for bench.FlsEngine (injected with FLS_BENCH_ENGINE=tests/fake_bench_engine.py:
FakeEngine) so tests/test_bench_cpu.py can drive bench.py's multi-rank contract -- spawn under
torch.distributed.run, one device per rank, barrier + max-over-ranks timing, one JSON line --
without a GPU.  Rank r's step sleeps (1 + r) ms, so the max over ranks is rank N-1's time.
FAKE_GPUS: devices the fake node has; FAKE_SAME_DEVICE=1: every rank reports the same device."""
import os
import time


class FakeEngine:
    backend = "gloo"

    @staticmethod
    def device_count():
        return int(os.environ.get("FAKE_GPUS", "8"))

    def __init__(self, args, world, rank, local):
        self.args, self.world, self.rank, self.local = args, world, rank, local
        self.entries_total = 1_000_000 * world
        self.steps_done = 0

    def device_id(self):
        return "fake-gpu-0" if os.environ.get("FAKE_SAME_DEVICE") == "1" else f"fake-gpu-{self.local}"

    def coll_device(self):
        return "cpu"

    def step(self):
        time.sleep(1e-3 * (1 + self.rank))
        self.steps_done += 1

    def sync(self):
        pass

    def begin_timed(self):
        pass

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        return 1e3 * (time.perf_counter() - self.t0)

    def end_timed(self):
        pass

    def kernel_report(self, steps):
        ms = 1.0 + self.rank
        return {"achieved": 8e6 / (ms / 1e3) / 1e9, "bytes_per_step": 8e6, "kernel_ms_per_step": ms,
                "kernel_ms_avg": ms, "launches": steps, "entries_per_s": 1e6 / (ms / 1e3)}

    def report(self, steps, ms_step, per_rank, n_gpus):
        return {"dtype": "f64", "config": {"workload": "fake", "ranks_reported": len(per_rank)},
                "roofline": {"bound": "hbm", "per_rank": per_rank}, "gpu_launches": steps,
                "clocks": {}}

    def extras(self, args):
        return {"warmup_and_steps_done_rank0": self.steps_done}

    def close(self):
        pass
