"""GPU check + timing of the tensor-core Prefill GEMM (csrc/prefill_gemm.cu) against torch float64 / cuBLAS.

    python tools/prefill_check.py [quick]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2605_11581_b200 import prefill as P  # noqa: E402


def planes_of(x, parts):
    hi = x.to(torch.bfloat16)
    if parts == 1:
        return hi[None].contiguous()
    lo = (x - hi.float()).to(torch.bfloat16)
    return torch.stack((hi, lo)).contiguous()


def check(T, K, N, parts, epi, tile_n=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, K, device="cuda", generator=g)
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    xp = planes_of(x, parts)
    ref = xp.double().sum(0) @ w.double().T
    if epi == P.EPI_SWIGLU:
        blk = 64 if tile_n == 128 else 128
        I = N // 2
        r = ref.view(T, I // blk, 2, blk)
        gate, up = r[:, :, 0].reshape(T, I), r[:, :, 1].reshape(T, I)
        want = torch.nn.functional.silu(gate) * up
        out = torch.zeros(2, T, I, dtype=torch.bfloat16, device="cuda")
        P.gemm(xp, w, out, epilogue=epi, tile_n=tile_n)
        got = out.double().sum(0)
        tol = 2e-4
    elif epi == P.EPI_RESID:
        out = torch.randn(T, N, device="cuda", generator=g)
        want = out.double() + ref
        P.gemm(xp, w, out, epilogue=epi, tile_n=tile_n)
        got = out.double()
        tol = 2e-5
    else:
        bias = torch.randn(N, device="cuda", generator=g)
        want = ref + bias.double()
        out = torch.zeros(T, N, device="cuda")
        P.gemm(xp, w, out, bias=bias, tile_n=tile_n)
        got = out.double()
        tol = 2e-5
    torch.cuda.synchronize()
    err = (got - want).abs().max().item()
    scale = want.abs().max().item()
    ok = err <= tol * max(scale, 1.0) * 4
    print(f"T {T:5d} K {K:5d} N {N:6d} parts {parts} epi {epi} tile {tile_n:3d}: max err {err:.3e} (scale {scale:.2f}) {'ok' if ok else 'FAIL'}",
          flush=True)
    return ok


def bench(T, K, N, parts, epi=P.EPI_STORE, tile_n=0, iters=20, rounds=3):
    """Ours and cuBLAS alternate in the same process (the box's SM clock moves with its power state, so only
    adjacent measurements compare); medians over ``rounds``."""
    x = torch.randn(parts, T, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    if epi == P.EPI_SWIGLU:
        out = torch.zeros(parts, T, N // 2, dtype=torch.bfloat16, device="cuda")
    else:
        out = torch.zeros(T, N, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    ours, lib = [], []
    for _ in range(rounds):
        ours.append(timed(lambda: P.gemm(x, w, out, epilogue=epi, tile_n=tile_n)))
        lib.append(timed(lambda: torch.matmul(x[0], w.T)))
    ms, ms_lib = sorted(ours)[rounds // 2], sorted(lib)[rounds // 2]
    tf = 2.0 * T * K * N * parts / ms / 1e9
    print(f"bench T {T} K {K} N {N} planes {parts} epi {epi} tile {tile_n}: {ms:.3f} ms {tf:.0f} TFLOP/s | cuBLAS bf16 (1 plane, no epilogue) "
          f"{ms_lib:.3f} ms {2.0 * T * K * N / ms_lib / 1e9:.0f} TFLOP/s | per-plane time ratio {ms / parts / ms_lib:.2f}", flush=True)


if __name__ == "__main__":
    ok = True
    ok &= check(128, 64, 128, 1, P.EPI_STORE, 128)
    ok &= check(128, 256, 256, 1, P.EPI_STORE, 256)
    ok &= check(300, 1536, 2048, 2, P.EPI_STORE)
    ok &= check(300, 1536, 2048, 2, P.EPI_STORE, 128)
    ok &= check(1000, 8960, 1536, 2, P.EPI_RESID)
    ok &= check(77, 192, 328, 1, P.EPI_RESID, 128)
    ok &= check(520, 1536, 2560, 2, P.EPI_SWIGLU, 256)
    ok &= check(130, 512, 1024, 1, P.EPI_SWIGLU, 128)
    ok &= check(2048, 3584, 4608, 2, P.EPI_STORE)
    for T in (256, 300, 77, 2048):
        ok &= check(T, 256, 256, 1, P.EPI_STORE, 512)
        ok &= check(T, 1536, 2048, 2, P.EPI_STORE, 512)
        ok &= check(T, 1536, 1320, 1, P.EPI_RESID, 512)
        ok &= check(T, 512, 2560, 2, P.EPI_SWIGLU, 512)
    ok &= check(4096, 3584, 3584, 1, P.EPI_RESID, 512)
    ok &= check(4096, 1536, 17920, 1, P.EPI_SWIGLU, 512)
    print("ALL OK" if ok else "FAILED", flush=True)
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        sys.exit(0 if ok else 1)
    for parts in (1, 2):
        for tile in (256, 512):
            bench(4096, 3584, 4608, parts, tile_n=tile)
            bench(4096, 3584, 3584, parts, P.EPI_RESID, tile)
            bench(4096, 3584, 37888, parts, P.EPI_SWIGLU, tile)
            bench(4096, 18944, 3584, parts, P.EPI_RESID, tile)
            bench(4096, 1536, 2048, parts, tile_n=tile)
            bench(4096, 1536, 17920, parts, P.EPI_SWIGLU, tile)
            bench(4096, 8960, 1536, parts, P.EPI_RESID, tile)
    sys.exit(0 if ok else 1)
