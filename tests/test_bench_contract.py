"""bench.py's reference arm (the oracle on host cores) prints one contract JSON line and
exits 0 on a CPU-only box; its other ranks exit 0 without output."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_line():
    r = _run({}, "--steps", "2", "--warmup", "1", "--cpu-seconds", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["unit"] == "coeffs/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("n15_dense_general")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_self_spawn_without_torchrun():
    """`bench.py --gpus 2` with no torchrun environment relaunches itself under
    torch.distributed.run with one rank per GPU (here --dry-run stops every rank before CUDA)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["master_addr"] == "127.0.0.1" for d in lines)


def test_spawn_command_and_combined_roofline():
    sys.path.insert(0, ROOT)
    import bench

    cmd = bench.spawn_cmd(8, ["--gpus", "8", "--steps", "3"], 29500)
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=8" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "8", "--steps", "3"]
    # n = 15 over 8 GPUs: 2^27 coefficients per rank, 32 B each through HBM, 7/8 of the
    # rank's 2 GiB shard over NVLink (4.30 GB and 1.88 GB)
    r = bench.combined_roofline(15, 8, 4.0, 6532.9, 700.0)
    assert r["hbm_bytes_per_rank"] == 32 * 2 ** 27 and r["a2a_bytes_sent_per_rank"] == 16 * 2 ** 27 * 7 // 8
    t_hbm = 32 * 2 ** 27 / 6532.9e9 * 1e3
    t_a2a = 16 * 2 ** 27 * 7 / 8 / 700e9 * 1e3
    assert abs(r["t_hbm_ms"] - t_hbm) < 1e-12 and abs(r["t_a2a_ms"] - t_a2a) < 1e-12
    assert abs(r["roofline_ms"] - (t_hbm + t_a2a)) < 1e-12
    assert abs(r["frac"] - (t_hbm + t_a2a) / 4.0) < 1e-12
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    one = bench.combined_roofline(15, 1, 8.0, 6532.9, 1.0)
    assert one["t_a2a_ms"] == 0.0 and one["bound"] == "hbm"
