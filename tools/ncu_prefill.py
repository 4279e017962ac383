"""ncu target: a few launches of the Prefill GEMM (Qwen2.5-7B shapes, T = 4096).  usage: ncu_prefill.py [planes]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import prefill as P

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T, H, I = 4096, 3584, 18944
x = torch.randn(parts, T, H, device="cuda").to(torch.bfloat16)
wgu = (torch.randn(2 * I, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
wd = (torch.randn(H, I, device="cuda") / I ** 0.5).to(torch.bfloat16)
act = torch.zeros(parts, T, I, dtype=torch.bfloat16, device="cuda")
h = torch.zeros(T, H, device="cuda")
for _ in range(2):
    P.gemm(x, wgu, act, epilogue=P.EPI_SWIGLU)
    P.gemm(act, wd, h, epilogue=P.EPI_RESID)
torch.cuda.synchronize()
