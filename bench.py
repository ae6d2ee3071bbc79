#!/usr/bin/env python
"""bench.py -- Pauli-coefficient throughput of the B200 path (BASELINE.json metric).

Default workload (N=1): dense general complex128 n=15 (32768 x 32768, 16 GiB),
seed 4 -- BASELINE.json configs[4], the configuration the metric
"Pauli coeffs/s + HBM GB/s, dense complex128 n=15/16 at 1/2/4/8 B200" is quoted on.
A step = one full decomposition (all 4^15 coefficients) of the HBM-resident input;
for N > 1 the step is the NCCL all-to-all (row blocks -> X-mask shards) plus the
per-rank decomposition (strong scaling: n fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 15] [--impl reference]

Prints ONE JSON line on rank 0.  The inputs (16 GiB) exceed the 126 MB L2, so no
flush is needed between timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Pauli coeffs/s + HBM GB/s, dense complex128 n=15/16 at 1/2/4/8 B200"
UNIT = "coeffs/s"
SEED = 4  # BASELINE.json configs[4]


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--n", type=int, default=15)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=12)  # steady state: fill and drain amortised
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                   help="N > 1: NCCL all-to-all then per-rank decomposition, or the fused "
                        "peer-pull kernel (TMA loads of the owners' row blocks over NVLink)")
    return p.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _profile_traffic(n):
    """dram bytes per launch of the fused kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        k = d.get("fused_kernel", {}).get(f"n{n}")
        return float(k["dram_bytes_per_launch"]) if k else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(n, seconds, variant=0):
    """The oracle as it stands, on the host cores, on a bounded sample of the same
    workload: coefficients of the n=15 seed-4 matrix at seeded random strings, with
    the entries generated on the fly by the host input module (the matrix is a
    function; materialising 16 GiB on the host is not part of it)."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(12345)
    threads = oracle.threads()
    batch = max(threads, 8)
    done, t0 = 0, time.perf_counter()
    elapsed = 0.0
    while elapsed < seconds:
        qs = rng.integers(0, 4 ** n, batch, dtype=np.uint64)
        oracle.coeffs_generated(n, SEED, variant, qs)
        done += batch
        elapsed = time.perf_counter() - t0
    return {"value": done / elapsed, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{done} seeded-random coefficients of the n={n} seed-{SEED} matrix "
                      f"(entries generated on the fly), {elapsed:.1f} s",
            "coefficients": done, "seconds": elapsed}


def run_reference(a):
    """The reference arm: the oracle (there is no reference code, the reference is a paper)
    timed on the host cores -- W untimed warm-up steps, then exactly K timed steps, each a
    bounded sample of the workload (about cpu_seconds / K seconds of oracle work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per = max(0.5, a.cpu_seconds / max(1, a.steps))
    for _ in range(max(0, a.warmup)):
        cpu_baseline(a.n, min(per, 0.5))
    runs = [cpu_baseline(a.n, per) for _ in range(max(1, a.steps))]
    done = sum(r["coefficients"] for r in runs)
    secs = sum(r["seconds"] for r in runs)
    v = done / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
        "steps": len(runs), "warmup": max(0, a.warmup), "ms_per_step": secs * 1e3 / len(runs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"n{a.n}_dense_general_seed{SEED}", "n": a.n,
                   "structure": "general", "seed": SEED},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": runs[0]["cores"], "kind": "oracle",
                         "sample": f"{done} seeded-random coefficients of the n={a.n} seed-{SEED} "
                                   f"matrix (entries generated on the fly) in {len(runs)} steps, "
                                   f"{secs:.1f} s"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist

    import paper_2403_11644_b200 as ptdr
    from paper_2403_11644_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        if a.gpus > 1:
            raise SystemExit(f"--gpus {a.gpus} needs torchrun with {a.gpus} ranks (WORLD_SIZE={world})")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = a.n
    N = 1 << n
    coeffs_total = 1 << (2 * n)
    stream = torch.cuda.current_stream()

    # ---- inputs resident in HBM (generator kernel, row a1; timed separately) ----------
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    if world == 1:
        A = ptdr.generate_dense(n, SEED, "general", device=dev)
        out = torch.empty(coeffs_total, dtype=torch.complex128, device=dev)
        ws = ptdr.alloc_workspace(n, "general", 1, dev)
    elif a.exchange == "peer":
        shard = ptdr.generate_dense(n, SEED, "general", row0=rank * (N // world), nrows=N // world, device=dev)
        out = torch.empty(coeffs_total // world, dtype=torch.complex128, device=dev)
        ws = ptdr.alloc_workspace(n, "general", world, dev)
    else:
        send = ptdr.generate_sendblocks(n, SEED, rank, world, device=dev)
        recv = torch.empty_like(send)
        out = torch.empty(coeffs_total // world, dtype=torch.complex128, device=dev)
        ws = ptdr.alloc_workspace(n, "general", world, dev)
    g1.record(stream)
    torch.cuda.synchronize()
    gen_ms = g0.elapsed_time(g1)
    peer_ptrs, peer_close = None, None
    if world > 1 and a.exchange == "peer":
        peer_ptrs, peer_close = pdist.open_peer_shards(shard)
        dist.barrier()

    ev_kernel = []
    ev_xchg = []

    def step(record):
        if world == 1:
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            ptdr.decompose(A, "general", out=out, workspace=ws, stream=stream)
            if record:
                e1.record(stream)
                ev_kernel.append((e0, e1))
        elif peer_ptrs is not None:
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            pdist.decompose_peer_sharded(shard, n, peer_ptrs, out=out, workspace=ws, stream=stream)
            if record:
                e1.record(stream)
                ev_kernel.append((e0, e1))
        else:
            if record:
                x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                x0.record(stream)
            pdist.exchange(send, None, recv)
            if record:
                x1.record(stream)
                ev_xchg.append((x0, x1))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            ptdr.decompose_xshard(recv.view(N, N // world), n, rank, world, out=out, workspace=ws,
                                  stream=stream)
            if record:
                e1.record(stream)
                ev_kernel.append((e0, e1))
        return ptdr.last_launch_count()

    for _ in range(max(a.warmup, 0)):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    launches = 0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record(stream)
    for _ in range(a.steps):
        launches += step(True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    elapsed_ms = t0.elapsed_time(t1)
    kern_ms = [e0.elapsed_time(e1) for e0, e1 in ev_kernel]
    xmean = statistics.mean([x0.elapsed_time(x1) for x0, x1 in ev_xchg]) if ev_xchg else 0.0
    if world > 1:
        tt = torch.tensor([elapsed_ms, statistics.mean(kern_ms), xmean], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms, kmean, xmean = tt.tolist()
    else:
        kmean = statistics.mean(kern_ms)
    ms_per_step = elapsed_ms / a.steps
    value = coeffs_total / (ms_per_step * 1e-3)

    # Parseval of the last step's output (cheap property check at full size)
    def sumsq(t):
        flat = torch.view_as_real(t.reshape(-1))
        tot = 0.0
        for i in range(0, flat.shape[0], 1 << 26):
            c = flat[i:i + (1 << 26)]
            tot += torch.sum(c * c).item()
        return tot

    if world == 1:
        lhs = sumsq(out)
        rhs = sumsq(A) / N
        parseval = abs(lhs - rhs) / rhs
    else:
        parseval = None

    # ---- roofline of the dominant kernel (the fused gather+WHT kernel) -----------------
    peak, peak_kind = _peaks()
    coeffs_per_rank = coeffs_total // world
    alg_bytes = 32 * coeffs_per_rank              # 16 B read + 16 B written per coefficient
    achieved = alg_bytes / (kmean * 1e-3) / 1e9
    traffic = _profile_traffic(n) if world == 1 else None

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"n{n}_dense_general_seed{SEED}", "n": n,
                       "structure": "general", "seed": SEED, "coefficients": coeffs_total,
                       "input_bytes": 16 * coeffs_total,
                       "l2": "inputs 16 GiB >> 126 MB L2 (no flush needed)",
                       "parallelism": "single GPU" if world == 1 else
                       (f"X-mask shards over {world} GPUs, fused peer-pull (TMA over NVLink)"
                        if peer_ptrs is not None else
                        f"X-mask shards over {world} GPUs, 1 NCCL all-to-all")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": "dense_pipe_kernel (PTDR_PIPE_CFG=%s)" % os.environ.get("PTDR_PIPE_CFG", "default"),
                         "kernel_ms": kmean, "algorithmic_bytes_per_launch": alg_bytes,
                         "hbm_passes": 1, "l2_round_trips": 1,
                         "note": "32 B/coefficient (16 B read of A + 16 B write); the partial "
                                 "transforms make one round trip through an L2-resident scratch, "
                                 "whose traffic alone (no arithmetic) takes 6.75-7.3 ms at n=15 "
                                 "(profiles/r01/micro/roundtrip_bench.txt; DESIGN.md section 7)"},
            "hbm_gbs_step": 32 * coeffs_total / (ms_per_step * 1e-3) / 1e9 / world,
            "gpu_launches": launches,
            "nvlink": (None if not ev_xchg else {
                "exchange_ms": xmean,
                "bytes_sent_per_rank": 16 * coeffs_total // world * (world - 1) // world,
                "gbs_per_rank": 16 * coeffs_total // world * (world - 1) // world / (xmean * 1e-3) / 1e9,
                "peak_per_direction_gbs": 770.0, "peak_kind": "measured peer copy (B200_PROFILING.md)"}),
            "generator_ms": gen_ms,
            "parseval_rel": parseval,
            "clocks": clk,
        }

    # ---- end to end through the public host API (rank 0, N == 1) ------------------------
    # HostPlan (ptdr_plan_*): every step uploads the step's matrix from pinned host memory,
    # decomposes it on the device and downloads all 4^n coefficients into pinned host
    # memory; with two device slots the upload of step k+1 overlaps the download of step k.
    if world == 1 and not a.no_e2e:
        def e2e_single():
            nonlocal A, ws
            del ws
            torch.cuda.empty_cache()
            import numpy as np

            host_in = torch.empty((N, N), dtype=torch.complex128, pin_memory=True)
            host_in.copy_(A)
            del A
            torch.cuda.empty_cache()
            host_out = [torch.empty(coeffs_total, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
            hin = host_in.numpy()
            houts = [h.numpy() for h in host_out]
            K = max(2, a.e2e_steps)
            with ptdr.HostPlan(n, "general", depth=2) as plan:
                plan.decompose_async(hin, houts[0])          # warm-up (allocations, module load)
                plan.wait()
                s0 = time.perf_counter()
                for k in range(K):
                    plan.decompose_async(hin, houts[k % 2])
                plan.wait()
                e2e_s = (time.perf_counter() - s0) / K
                e2e_launches = plan.launch_count() * K
            # the streamed result must equal the device-timed one (same kernels, same input)
            idx = torch.from_numpy(np.random.default_rng(7).integers(0, coeffs_total, 1 << 16))
            same = bool(torch.equal(host_out[(K - 1) % 2][idx], out[idx.to(dev)].cpu()))
            line["e2e"] = {"value": coeffs_total / e2e_s, "unit": UNIT,
                           "h2d_bytes_per_step": 16 * coeffs_total, "d2h_bytes_per_step": 16 * coeffs_total,
                           "steps": K, "s_per_step": e2e_s, "gpu_launches": e2e_launches,
                           "matches_device_result": same,
                           "api": "ptdr_plan_decompose_host_async, depth 2 (pinned host buffers)"}
            del host_in, host_out, hin, houts

        try:
            e2e_single()
        except Exception as exc:  # never lose the bench line over the e2e leg (e.g. pinned memory)
            line["e2e"] = {"error": repr(exc)[:200]}

    # ---- end to end at N > 1: every rank uploads its row block from pinned host memory,
    # the step runs (exchange + decomposition, or the peer-pull kernel), and every rank
    # downloads its coefficient shard; wall time between barriers, max over ranks.
    if world > 1 and not a.no_e2e:
        try:
            src = shard if peer_ptrs is not None else send
            host_in = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
            host_in.copy_(src)
            host_out = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            K = max(2, a.e2e_steps)
            torch.cuda.synchronize()
            dist.barrier()
            s0 = time.perf_counter()
            for _ in range(K):
                src.copy_(host_in, non_blocking=True)
                if peer_ptrs is not None:
                    torch.cuda.synchronize()
                    dist.barrier()          # every shard uploaded before any rank reads it
                    pdist.decompose_peer_sharded(shard, n, peer_ptrs, out=out, workspace=ws, stream=stream)
                    torch.cuda.synchronize()
                    dist.barrier()          # every rank done reading before the next upload
                else:
                    pdist.decompose_sharded(send, n, out=out, recv=recv, workspace=ws, stream=stream)
                host_out.copy_(out, non_blocking=True)
            torch.cuda.synchronize()
            dist.barrier()
            tt = torch.tensor([(time.perf_counter() - s0) / K], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = tt.item()
            if rank == 0:
                line["e2e"] = {"value": coeffs_total / e2e_s, "unit": UNIT,
                               "h2d_bytes_per_step": 16 * coeffs_total,
                               "d2h_bytes_per_step": 16 * coeffs_total, "steps": K, "s_per_step": e2e_s,
                               "api": "pinned host row blocks -> " + ("decompose_peer_sharded" if peer_ptrs
                                                                     is not None else "decompose_sharded")
                                      + " -> pinned host shards (all ranks)"}
            del host_in, host_out
        except Exception as exc:  # never lose the bench line over the e2e leg
            if rank == 0:
                line["e2e"] = {"error": repr(exc)[:200]}

    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb = cpu_baseline(n, a.cpu_seconds)
        line["cpu_baseline"] = {k: v for k, v in cb.items() if k not in ("coefficients", "seconds")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if peer_close is not None:
            torch.cuda.synchronize()
            dist.barrier()
            peer_close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
