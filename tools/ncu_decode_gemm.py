"""ncu target: the decode-sized (split-K, atomic) GEMMs of one Qwen2.5-1.5B layer at batch 8."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import prefill as P

B, H, I = 8, 1536, 8960
x = torch.randn(2, B, H, device="cuda").to(torch.bfloat16)
a = torch.randn(2, B, I, device="cuda").to(torch.bfloat16)
wqkv = (torch.randn(2048, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
wgu = (torch.randn(2 * I, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
wd = (torch.randn(H, I, device="cuda") / I ** 0.5).to(torch.bfloat16)
qkv = torch.zeros(B, 2048, device="cuda")
gu = torch.zeros(B, 2 * I, device="cuda")
h = torch.zeros(B, H, device="cuda")
for _ in range(3):
    P.gemm(x, wqkv, qkv, epilogue=P.EPI_ATOMIC)
    P.gemm(x, wgu, gu, epilogue=P.EPI_ATOMIC)
    P.gemm(a, wd, h, epilogue=P.EPI_ATOMIC)
torch.cuda.synchronize()
