"""bench.py contract pieces that run without a GPU: the --impl reference arm (the CPU oracle,
tier rules) prints one JSON line at N=1 and, under torchrun with 2 ranks (gloo-free: the
reference arm needs no process group), only rank 0 prints."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_single():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--ref-rows", "32", "--workload", "c3_poisson5d"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    j = lines[0]
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "entries/s"
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "oracle"
    assert j["steps"] == 2 and j["warmup"] == 1


def test_reference_arm_two_ranks_prints_once():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_port()), "bench.py", "--impl", "reference", "--gpus", "2", "--steps",
                        "1", "--warmup", "0", "--ref-rows", "16", "--workload", "c2_poisson2d"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_clock_sampler_keeps_timed_window_and_flags_reasons():
    import datetime
    sys.path.insert(0, ROOT)
    import bench
    c = bench.ClockSampler(0)
    t = datetime.datetime(2026, 1, 1, 12, 0, 0)

    def row(sec, mhz, power_cap="Not Active", thermal="Not Active"):
        return (t + datetime.timedelta(seconds=sec),
                ["0", str(mhz), "1965", "500.0", "0x0", "Not Active", "Not Active", thermal, power_cap])
    c.rows = [row(0.0, 1965), row(1.0, 1500, "Active"), row(1.1, 1600, "Active"), row(3.0, 1965)]
    c.t0, c.t1 = t + datetime.timedelta(seconds=0.5), t + datetime.timedelta(seconds=2)
    out = c.stop()
    assert out["window"] == "timed region" and out["samples"] == 2
    assert out["sm_mhz"] == 1550 and out["sm_max_mhz"] == 1965 and out["reasons"] == ["sw_power_cap"]
    c.t0, c.t1 = t + datetime.timedelta(seconds=5), t + datetime.timedelta(seconds=6)
    c.rows.append(row(3.5, 1200, thermal="Active"))
    out = c.stop()                       # nothing inside the window: every sample counts
    assert out["window"] == "sampler lifetime" and out["samples"] == 5
    assert out["reasons"] == ["sw_power_cap", "sw_thermal_slowdown"]


def _bench(args, env_extra, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra)
    return subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout, env=env)


FAKE = {"FLS_BENCH_ENGINE": "tests/fake_bench_engine.py:FakeEngine"}


def test_gpus_flag_spawns_one_rank_per_device():
    """`bench.py --gpus 2` without a launcher starts 2 ranks itself (torch.distributed.run);
    exactly one JSON line, n_gpus = distinct devices = 2, time = max over ranks"""
    r = _bench(["--gpus", "2", "--steps", "5", "--warmup", "3"], dict(FAKE, FAKE_GPUS="2"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    j = lines[0]
    assert j["n_gpus"] == 2 and j["ranks"] == 2 and j["steps"] == 5 and j["warmup"] == 3
    assert j["ms_per_step"] >= 2.0                    # rank 1 sleeps 2 ms per step: the max
    assert j["value"] == 2_000_000 / (j["ms_per_step"] / 1e3)
    assert j["config"]["ranks_reported"] == 2 and j["warmup_and_steps_done_rank0"] == 8


def test_gpus_flag_fails_loudly_without_enough_devices():
    r = _bench(["--gpus", "4", "--steps", "1"], dict(FAKE, FAKE_GPUS="2"))
    assert r.returncode == 2 and "needs 4 GPUs" in r.stderr and not _json_lines(r.stdout)
    # the real engine on this GPU-less box
    r = _bench(["--gpus", "2", "--steps", "1"], {})
    assert r.returncode == 2 and "needs 2 GPUs" in r.stderr


def test_world_size_must_match_gpus_and_devices_must_be_distinct():
    r = _bench(["--gpus", "1", "--steps", "1"], dict(FAKE, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
    r = _bench(["--gpus", "2", "--steps", "2", "--warmup", "3"],
               dict(FAKE, FAKE_GPUS="2", FAKE_SAME_DEVICE="1"))
    assert r.returncode != 0 and "share 1 device" in r.stderr and not _json_lines(r.stdout)


def test_launcher_at_world_size_one_runs_the_collective_path():
    """under torchrun with one rank the process group is created too (the timing collectives
    then run exactly as at N > 1)"""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(FAKE, FAKE_GPUS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1", "--master-port",
                        str(_port()), "bench.py", "--gpus", "1", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 1 and lines[0]["ranks"] == 1
