#!/usr/bin/env python
"""A/B of the Prefill GEMM's tile walk order (adamk_prefill_set_walk): down-projection shapes and the whole 1.5B pass."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import prefill as P

lib = P._lib()


def timed(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


T = 4096
for name, H, I in (("qwen2.5-1.5b", 1536, 8960), ("qwen2.5-7b", 3584, 18944)):
    act = torch.randn(1, T, I, device="cuda").to(torch.bfloat16)
    wd = (torch.randn(H, I, device="cuda") / I ** 0.5).to(torch.bfloat16)
    h = torch.zeros(T, H, device="cuda")
    xb = act[0]
    ref = timed(lambda: torch.matmul(xb, wd.t()))
    row = []
    for mode in (0, 1, -1):
        lib.adamk_prefill_set_walk(mode)
        row.append(timed(lambda: P.gemm(act, wd, h, epilogue=P.EPI_RESID)))
    lib.adamk_prefill_set_walk(-1)
    fl = 2 * T * H * I / 1e9
    print(f"{name} down T={T}: token-fastest {row[0]*1e3:.1f} us ({fl/row[0]:.0f} TF/s) | column-fastest {row[1]*1e3:.1f} us ({fl/row[1]:.0f}) | "
          f"auto {row[2]*1e3:.1f} us | cuBLAS bf16 {ref*1e3:.1f} us ({fl/ref:.0f})")
