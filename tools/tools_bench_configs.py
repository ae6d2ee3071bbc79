"""Time every BASELINE.json configuration on one GPU (CUDA events, device-resident input).

Prints one JSON line per configuration with ms, coefficients/s and the achieved
algorithmic HBM bandwidth (bytes per coefficient as in DESIGN.md section 7):
dense 32 B, Hermitian/real-symmetric 24 B (upper triangle read + output), diagonal
32 B, tridiagonal (band bytes + output bytes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2403_11644_b200 as ptdr  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6534.8


def time_it(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for e0, e1 in ev:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    return t[len(t) // 2]


def oracle_rate(fn, n_out, seconds=2.0):
    """The CPU oracle timed beside the kernel (all host cores): coefficients/s on seeded
    random strings of the same workload, bounded to ~`seconds`."""
    import time

    import numpy as np

    import oracle

    rng = np.random.default_rng(3)
    batch = max(oracle.threads(), 8)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        fn(rng.integers(0, n_out, batch, dtype=np.uint64))
        done += batch
    rate = done / (time.perf_counter() - t0)
    return {"oracle_coeffs_per_s": rate, "oracle_cores": oracle.threads(),
            "oracle_projected_full_s": n_out / rate}


def dense(name, n, seed, variant):
    A = ptdr.generate_dense(n, seed, variant, device="cuda")
    out = torch.empty(1 << (2 * n), dtype=torch.complex128, device="cuda")
    ws = ptdr.alloc_workspace(n, variant, 1, "cuda")
    ms = time_it(lambda: ptdr.decompose(A, variant, out=out, workspace=ws))
    coeffs = 1 << (2 * n)
    graph_ms = None
    if n <= 13:
        # launch-bound sizes: the same call captured once in a CUDA graph and replayed
        # (device time without the Python/ctypes launch overhead)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ptdr.decompose(A, variant, out=out, workspace=ws, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ptdr.decompose(A, variant, out=out, workspace=ws, stream=s)
        reps = 20
        graph_ms = time_it(lambda: [g.replay() for _ in range(reps)]) / reps
    bpc = 32 if variant == "general" else 24
    gbs = bpc * coeffs / (ms * 1e-3) / 1e9
    import oracle
    import ptdr_inputs

    vnum = ptdr_inputs.VARIANTS.get(variant, variant)
    orc = oracle_rate(lambda qs: oracle.coeffs_generated(n, seed, vnum, qs), coeffs)
    print(json.dumps({"config": name, "n": n, "structure": variant, "ms": ms,
                      "coeffs_per_s": coeffs / (ms * 1e-3), "alg_bytes_per_coeff": bpc,
                      "hbm_gbs": gbs, "frac_of_measured": gbs / PEAK, "graph_replay_ms": graph_ms,
                      "graph_coeffs_per_s": coeffs / (graph_ms * 1e-3) if graph_ms else None, **orc}),
          flush=True)
    del A, out, ws
    torch.cuda.empty_cache()


def band(name, n, seed, variant):
    B = ptdr.generate_band(n, seed, variant, device="cuda")
    out = torch.empty(ptdr.output_count(n, variant), dtype=torch.complex128, device="cuda")
    ws = ptdr.alloc_workspace(n, variant, 1, "cuda")
    ms = time_it(lambda: ptdr.decompose(B, variant, out=out, workspace=ws))
    coeffs = out.numel()
    alg = (B.numel() + out.numel()) * 16
    gbs = alg / (ms * 1e-3) / 1e9
    import numpy as np

    import oracle
    import ptdr_inputs
    from paper_2403_11644_b200 import q_of

    if variant in ("tridiagonal", "hermitian_tridiagonal"):
        sub, main, sup = ptdr_inputs.band(n, seed, "tridiagonal")

        def orc_fn(idx):
            qs = np.array([q_of((1 << int(b)) - 1, int(z), n) for b, z in zip(idx >> n, idx & ((1 << n) - 1))],
                          dtype=np.uint64)
            return oracle.coeffs_tridiagonal(sub, main, sup, qs)
    else:
        d = ptdr_inputs.band(n, seed, "diagonal")

        def orc_fn(idx):
            return oracle.coeffs_diagonal(d, np.array([q_of(0, int(z), n) for z in idx], dtype=np.uint64))
    orc = oracle_rate(orc_fn, coeffs, seconds=3.0)
    print(json.dumps({"config": name, "n": n, "structure": variant, "ms": ms,
                      "coeffs_per_s": coeffs / (ms * 1e-3), "alg_bytes": alg, "hbm_gbs": gbs,
                      "frac_of_measured": gbs / PEAK, "launches": ptdr.last_launch_count(), **orc}),
          flush=True)
    # 8 GPUs, replicated band + z-sharded output: ranks are independent (no communication),
    # so the 8-GPU step time is the max over ranks of each rank's own time (ranks 0 and 7 here)
    world = 8
    outl = torch.empty(ptdr.output_count(n, variant) // world, dtype=torch.complex128, device="cuda")
    wsl = ptdr.alloc_workspace(n, variant, world, "cuda")
    ms8 = max(time_it(lambda: ptdr.decompose_zshard(B, variant, r, world, out=outl, workspace=wsl))
              for r in (0, world - 1))
    print(json.dumps({"config": name + "_8gpu_zshard", "n": n, "structure": variant, "ms_per_rank": ms8,
                      "coeffs_per_s_total": coeffs / (ms8 * 1e-3),
                      "alg_bytes_per_rank": (B.numel() + out.numel() // world) * 16,
                      "hbm_gbs_per_rank": (B.numel() + out.numel() // world) * 16 / (ms8 * 1e-3) / 1e9}),
          flush=True)
    del B, out, ws, outl, wsl
    torch.cuda.empty_cache()


def band_s(name, n, s):
    """(2s+1)-band: seeded N(0,1) diagonals, all nonzero-X-mask blocks."""
    g = torch.Generator(device="cuda").manual_seed(5)
    diags = torch.complex(torch.randn(2 * s + 1, 1 << n, generator=g, device="cuda", dtype=torch.float64),
                          torch.randn(2 * s + 1, 1 << n, generator=g, device="cuda", dtype=torch.float64))
    nb = len(ptdr.band_xmasks(n, s))
    out = torch.empty(nb << n, dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(ptdr.lib().ptdr_band_workspace_bytes(n, s)), dtype=torch.uint8, device="cuda")
    ms = time_it(lambda: ptdr.decompose_band(diags, s, out=out, workspace=ws))
    alg = (diags.numel() + out.numel()) * 16
    print(json.dumps({"config": name, "n": n, "s": s, "blocks": nb, "ms": ms,
                      "coeffs_per_s": out.numel() / (ms * 1e-3), "alg_bytes": alg,
                      "hbm_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_measured": alg / (ms * 1e-3) / 1e9 / PEAK,
                      "launches": ptdr.last_launch_count()}), flush=True)
    del diags, out, ws
    torch.cuda.empty_cache()


def anti(name, n):
    g = torch.Generator(device="cuda").manual_seed(6)
    a = torch.complex(torch.randn(1 << n, generator=g, device="cuda", dtype=torch.float64),
                      torch.randn(1 << n, generator=g, device="cuda", dtype=torch.float64))
    out = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    ms = time_it(lambda: ptdr.decompose(a, "anti_diagonal", out=out))
    alg = 32 * (1 << n)
    print(json.dumps({"config": name, "n": n, "ms": ms, "coeffs_per_s": (1 << n) / (ms * 1e-3),
                      "hbm_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_measured": alg / (ms * 1e-3) / 1e9 / PEAK,
                      "launches": ptdr.last_launch_count()}), flush=True)


def generated(name, n):
    """Matrix-free: entries computed in phase A, A never stored."""
    out = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(ptdr.lib().ptdr_generated_workspace_bytes(n, 1)), dtype=torch.uint8, device="cuda")
    ms = time_it(lambda: ptdr.decompose_generated(n, 4, out=out, workspace=ws), iters=5, warm=2)
    print(json.dumps({"config": name, "n": n, "ms": ms, "coeffs_per_s": 4 ** n / (ms * 1e-3),
                      "hbm_gbs_16B": 16 * 4 ** n / (ms * 1e-3) / 1e9,
                      "frac_of_measured_16B": 16 * 4 ** n / (ms * 1e-3) / 1e9 / PEAK,
                      "launches": ptdr.last_launch_count()}), flush=True)
    del out, ws
    torch.cuda.empty_cache()


def batched(name, n, batch):
    """Batched small matrices: one launch for the whole batch (amortises launch latency)."""
    A = torch.randn((batch, 1 << n, 1 << n), dtype=torch.complex128, device="cuda")
    out = torch.empty((batch, 4 ** n), dtype=torch.complex128, device="cuda")
    ms = time_it(lambda: ptdr.decompose_batched(A, "general", out=out))
    coeffs = batch * 4 ** n
    print(json.dumps({"config": name, "n": n, "batch": batch, "ms": ms, "coeffs_per_s": coeffs / (ms * 1e-3),
                      "hbm_gbs": 32 * coeffs / (ms * 1e-3) / 1e9,
                      "frac_of_measured": 32 * coeffs / (ms * 1e-3) / 1e9 / PEAK,
                      "launches": ptdr.last_launch_count()}), flush=True)
    del A, out
    torch.cuda.empty_cache()


def inverse(name, n):
    """Inverse transform: coefficients -> A, round trip checked."""
    A = ptdr.generate_dense(n, 4, "general", device="cuda")
    c = ptdr.decompose(A)
    B = torch.empty_like(A)
    ws = torch.empty(int(ptdr.lib().ptdr_reconstruct_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    ms = time_it(lambda: ptdr.reconstruct(c, out=B, workspace=ws))
    err = max(torch.max(torch.abs(A[i:i + 1024] - B[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    alg = 32 * 4 ** n
    print(json.dumps({"config": name, "n": n, "ms": ms, "coeffs_per_s": 4 ** n / (ms * 1e-3),
                      "hbm_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_measured": alg / (ms * 1e-3) / 1e9 / PEAK,
                      "round_trip_max_err": err, "launches": ptdr.last_launch_count()}), flush=True)
    del A, B, c, ws
    torch.cuda.empty_cache()


def inverse_layout(name, n, inplace_call):
    """Inverse transform from the matrix layout (ptdr_reconstruct_matrix_layout_async, MODE_INV
    pipeline at n >= 11), out of place or in place; round trip checked."""
    A = ptdr.generate_dense(n, 4, "general", device="cuda")
    M = ptdr.decompose_matrix_layout(A)
    ws = torch.empty(int(ptdr.lib().ptdr_reconstruct_matrix_layout_workspace_bytes(n)), dtype=torch.uint8,
                     device="cuda")
    if inplace_call:
        del A
        torch.cuda.empty_cache()
        src = M.clone()
        times = []
        for it in range(8):
            M.copy_(src)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ptdr.reconstruct_matrix_layout(M, workspace=ws, inplace=True)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[len(times) // 2]
        del src
        A = ptdr.generate_dense(n, 4, "general", device="cuda")
        B = M
    else:
        B = torch.empty_like(A)
        ms = time_it(lambda: ptdr.reconstruct_matrix_layout(M, out=B, workspace=ws))
    err = max(torch.max(torch.abs(A[i:i + 1024] - B[i:i + 1024])).item() for i in range(0, A.shape[0], 1024))
    alg = 32 * 4 ** n
    print(json.dumps({"config": name, "n": n, "in_place": inplace_call, "ms": ms, "coeffs_per_s": 4 ** n / (ms * 1e-3),
                      "hbm_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_measured": alg / (ms * 1e-3) / 1e9 / PEAK,
                      "round_trip_max_err": err, "launches": ptdr.last_launch_count()}), flush=True)
    del A, B, M, ws
    torch.cuda.empty_cache()


def xshard(name, n, world):
    """BASELINE configs[4] at G GPUs, per rank, kernel side: the X-mask shard decomposition
    one rank runs after its all-to-all (ranks 0 and G-1 emulated on this GPU; the exchange
    itself is timed in bench.py's N > 1 line)."""
    R = (1 << n) // world
    A = ptdr.generate_dense(n, 4, "general", device="cuda")
    V = A.view(world, R, world, R)
    ws = ptdr.alloc_workspace(n, "general", world, "cuda")
    out = torch.empty(4 ** n // world, dtype=torch.complex128, device="cuda")
    ms = 0.0
    for h in (0, world - 1):
        recv = torch.stack([V[g, :, g ^ h, :] for g in range(world)]).contiguous().view(1 << n, R)
        ms = max(ms, time_it(lambda: ptdr.decompose_xshard(recv, n, h, world, out=out, workspace=ws)))
        del recv
    coeffs = 4 ** n // world
    gbs = 32 * coeffs / (ms * 1e-3) / 1e9
    a2a = 16 * coeffs * (world - 1) // world
    print(json.dumps({"config": name, "n": n, "world": world, "ms_per_rank": ms, "coeffs_per_s_total": 4 ** n / (ms * 1e-3),
                      "hbm_gbs_per_rank": gbs, "frac_of_measured": gbs / PEAK, "a2a_bytes_sent_per_rank": a2a}),
          flush=True)
    del A, V, ws, out
    torch.cuda.empty_cache()


def inplace(name, n, seed):
    """BASELINE configs[4] "n=16 at 1 GPU in-place": ptdr_decompose_inplace_async overwrites A
    with its coefficients (matrix layout); A is regenerated before every timed call (the
    generator outside the timed region)."""
    A = ptdr.generate_dense(n, seed, "general", device="cuda")
    nb = int(ptdr.lib().ptdr_inplace_workspace_bytes(n, 0))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    times = []
    for it in range(8):
        ptdr.generate_dense(n, seed, "general", out=A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ptdr.decompose(A, "general", workspace=ws, inplace=True)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    ms = sorted(times)[len(times) // 2]
    coeffs = 1 << (2 * n)
    gbs = 32 * coeffs / (ms * 1e-3) / 1e9
    peak_gib = (16 * coeffs + nb) / 2 ** 30
    print(json.dumps({"config": name, "n": n, "structure": "general", "ms": ms, "coeffs_per_s": coeffs / (ms * 1e-3),
                      "alg_bytes_per_coeff": 32, "hbm_gbs": gbs, "frac_of_measured": gbs / PEAK,
                      "device_memory_gib": peak_gib}), flush=True)
    del A, ws
    torch.cuda.empty_cache()


def matrix_layout(name, n, seed):
    """The same transform out of place with the matrix-layout output (for comparison with
    the in-place call and the q-order one)."""
    A = ptdr.generate_dense(n, seed, "general", device="cuda")
    out = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(ptdr.lib().ptdr_inplace_workspace_bytes(n, 0)), dtype=torch.uint8, device="cuda")
    ms = time_it(lambda: ptdr.decompose_matrix_layout(A, "general", out=out, workspace=ws))
    coeffs = 1 << (2 * n)
    gbs = 32 * coeffs / (ms * 1e-3) / 1e9
    print(json.dumps({"config": name, "n": n, "structure": "general", "ms": ms, "coeffs_per_s": coeffs / (ms * 1e-3),
                      "alg_bytes_per_coeff": 32, "hbm_gbs": gbs, "frac_of_measured": gbs / PEAK}), flush=True)
    del A, out, ws
    torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    if "all" in which or "small" in which:
        dense("n6", 6, 0, "general")
        dense("n10a", 10, 1, "general")
        # the oracle's per-core rate: one thread, n = 10
        import subprocess
        r = subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_percore.py"),
                            "10"], env=dict(os.environ, OMP_NUM_THREADS="1"), capture_output=True, text=True)
        if r.returncode == 0:
            print(json.dumps({"config": "n10a_oracle_one_core", **json.loads(r.stdout.strip().splitlines()[-1])}),
                  flush=True)
        dense("n10b", 10, 1, "hermitian")
    if "all" in which or "n13" in which:
        dense("n13a", 13, 2, "hermitian")
        dense("n13b", 13, 2, "real_symmetric")
        dense("n13_general", 13, 2, "general")
    if "all" in which or "band" in which:
        band("n24tri", 24, 3, "tridiagonal")
        band("n24diag", 24, 3, "diagonal")
        band("n24tri_hermitian", 24, 3, "hermitian_tridiagonal")
    if "all" in which or "next" in which:
        anti("n24anti", 24)
        band_s("n24band_s2", 24, 2)
        band_s("n22band_s5", 22, 5)
        inverse("n15_inverse", 15)
        inverse_layout("n15_inverse_matrix_layout", 15, False)
        inverse_layout("n15_inverse_in_place", 15, True)
        batched("n6_batch16384", 6, 16384)
        batched("n10_batch64", 10, 64)
        generated("n15_matrix_free", 15)
    if "all" in which or "big" in which:
        dense("n15", 15, 4, "general")
        dense("n15_hermitian", 15, 4, "hermitian")
        dense("n16", 16, 4, "general")
    if "all" in which or "xshard" in which:
        xshard("n15_2gpu_xshard_kernel", 15, 2)
        xshard("n15_4gpu_xshard_kernel", 15, 4)
        xshard("n15_8gpu_xshard_kernel", 15, 8)
        xshard("n16_8gpu_xshard_kernel", 16, 8)
    if "inverse" in which:
        inverse("n15_inverse", 15)
        inverse_layout("n15_inverse_matrix_layout", 15, False)
        inverse_layout("n15_inverse_in_place", 15, True)
        inverse_layout("n16_inverse_in_place", 16, True)
    if "all" in which or "big" in which or "inplace" in which:
        inplace("n15_inplace", 15, 4)
        inplace("n16_inplace", 16, 4)
        matrix_layout("n15_matrix_layout", 15, 4)
        matrix_layout("n16_matrix_layout", 16, 4)
