#!/usr/bin/env python
"""Alternating A/B of the Prefill attention: this library's tcgen05 flash kernel (csrc/prefill_attn.cu, V^T included)
against torch's scaled_dot_product_attention (cuDNN / flash backend) on the same bf16 tensors.

    python tools/attn_bench.py [n_q] [n_kv] [D] [T ...]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.nn.functional as F
from paper_2605_11581_b200.prefill import _attn_ok, _lib, _ptr, _stream

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 28
nkv = int(sys.argv[2]) if len(sys.argv) > 2 else 4
D = int(sys.argv[3]) if len(sys.argv) > 3 else 128
Ts = [int(a) for a in sys.argv[4:]] or [4096, 16384]
lib = _lib()


def timed(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for T in Ts:
    q = torch.randn(nq, T, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(nkv, T, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(nkv, T, D, device="cuda").to(torch.bfloat16)
    ctx_pad = -(-T // 64) * 64
    vt = torch.empty(nkv, D, ctx_pad, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(1, T, nq * D, device="cuda", dtype=torch.bfloat16)

    def ours():
        _attn_ok(lib.adamk_prefill_vt(_ptr(v), nkv, D, T, T, ctx_pad, _ptr(vt), _stream()))
        _attn_ok(lib.adamk_prefill_attention(_ptr(q), _ptr(k), _ptr(vt), T, 0, nq, nkv, D, T, ctx_pad, _ptr(out), 1, _stream()))

    def lib_sdpa():
        return F.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True, enable_gqa=True)

    flops = 4.0 * nq * D * T * T / 2   # causal: half of QK^T and PV
    res = []
    for _ in range(3):   # alternate
        res.append((timed(ours), timed(lib_sdpa)))
    a = min(r[0] for r in res); b = min(r[1] for r in res)
    ref = lib_sdpa()[0].transpose(0, 1).reshape(T, nq * D).float()
    ours()
    torch.cuda.synchronize()
    err = (out[0].float() - ref).abs().max().item()
    print(f"n_q {nq} n_kv {nkv} D {D} T {T}: flash kernel {a:.3f} ms ({flops / a / 1e9:.0f} TFLOP/s)  |  library SDPA {b:.3f} ms "
          f"({flops / b / 1e9:.0f} TFLOP/s)  |  ratio ours/library {a / b:.2f}  |  max diff {err:.2e}", flush=True)
