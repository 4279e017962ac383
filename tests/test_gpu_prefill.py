"""Parity of the hand-written Prefill operators (include/adamk_prefill.h, through the C ABI) on a B200.

The tensor-core GEMM is checked against a float64 product of the same bf16 operands (the only difference is the
fp32 accumulation order inside the tensor cores: bound 4e-5 x the output scale) and the whole Prefill pass
against ``oracle.decode_ref.RefDecoder.prefill``: with two activation planes (hi + lo, 2^-17 relative) every KV
cache entry is within one bf16 ulp of the oracle's; > 99 % of layer 0 is bit-identical (measured 99.7 %), deeper
layers less (95 % in layer 1) because every one-ulp flip in a cached bf16 value perturbs what follows -- the decode
kernel's own fp32 path gives 99.98 % / 98.9 % against the oracle on the same prompt.
"""

import numpy as np
import pytest
import torch

from paper_2605_11581_b200.model_config import TINY, TINY_QWEN3, ModelConfig

pytestmark = pytest.mark.gpu

D128 = ModelConfig(name="test-d128", hidden=512, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=128,
                   intermediate=1280, vocab=4096)
D128_Q3 = ModelConfig(name="test-d128-q3", hidden=512, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128,
                      intermediate=1536, vocab=3000, qkv_bias=False, qk_norm=True, tied_embed=False)


def _planes(x, parts):
    hi = x.to(torch.bfloat16)
    if parts == 1:
        return hi[None].contiguous()
    return torch.stack((hi, (x - hi.float()).to(torch.bfloat16))).contiguous()


@pytest.mark.parametrize("T,K,N,parts,tile_n", [
    # tile_n: 128 / 256 = one CTA per 128 x tile_n tile, 512 = a CTA pair per 256 x 256 tile, 0 = the library's choice
    (128, 64, 128, 1, 128), (128, 256, 256, 1, 256), (1, 64, 8, 1, 128), (300, 1536, 2048, 2, 0), (300, 1536, 2048, 2, 128),
    (77, 192, 328, 1, 128), (77, 200, 328, 2, 256), (2048, 3584, 4608, 2, 0), (4096, 1536, 2048, 1, 0),
    (256, 256, 256, 1, 512), (300, 1536, 2048, 2, 512), (77, 200, 328, 1, 512), (4096, 1536, 2048, 1, 512), (1100, 512, 9728, 2, 512)])
def test_gemm_store_bias(T, K, N, parts, tile_n):
    from paper_2605_11581_b200 import prefill as P

    g = torch.Generator(device="cuda").manual_seed(T + K + N)
    x = torch.randn(T, K, device="cuda", generator=g)
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    xp = _planes(x, parts)
    want = xp.double().sum(0) @ w.double().T + bias.double()
    out = torch.full((T, N), float("nan"), device="cuda")
    P.gemm(xp, w, out, bias=bias, tile_n=tile_n)
    err = (out.double() - want).abs().max().item()
    assert err <= 4e-5 * max(1.0, want.abs().max().item()), err
    if parts == 2:   # two planes reproduce the fp32 activation: compare with the fp32-activation product
        exact = x.double() @ w.double().T + bias.double()
        assert (out.double() - exact).abs().max().item() <= 1e-4 * max(1.0, exact.abs().max().item())


@pytest.mark.parametrize("T,K,N,tile_n,epi", [(1100, 512, 1536, 0, "store"), (1100, 512, 1536, 128, "store"), (4096, 2048, 1536, 512, "resid"),
                                              (700, 256, 1024, 256, "swiglu"), (2100, 1024, 768, 0, "resid")])
def test_gemm_walk_orders_agree_bit_for_bit(T, K, N, tile_n, epi):
    """`adamk_prefill_set_walk`: token-block-fastest and tile-column-fastest walks assign the same tiles to different
    CTAs; every output element is computed by the same instructions, so the results are identical (whole tiles and the
    column slices of the last wave, one-CTA and CTA-pair kernels, every epilogue)."""
    from paper_2605_11581_b200 import prefill as P

    lib = P._lib()
    g = torch.Generator(device="cuda").manual_seed(T + N)
    xp = _planes(torch.randn(T, K, device="cuda", generator=g), 1)
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    base = torch.randn(T, N, device="cuda", generator=g)
    outs = []
    try:
        for mode in (0, 1, -1):
            lib.adamk_prefill_set_walk(mode)
            if epi == "swiglu":
                out = torch.zeros(1, T, N // 2, dtype=torch.bfloat16, device="cuda")
                P.gemm(xp, w, out, epilogue=P.EPI_SWIGLU, tile_n=tile_n)
            else:
                out = base.clone()
                P.gemm(xp, w, out, epilogue=P.EPI_RESID if epi == "resid" else P.EPI_STORE, tile_n=tile_n)
            outs.append(out)
    finally:
        lib.adamk_prefill_set_walk(-1)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    if epi != "swiglu":
        want = xp[0].double() @ w.double().T + (base.double() if epi == "resid" else 0)
        assert (outs[1].double() - want).abs().max().item() <= 4e-5 * max(1.0, want.abs().max().item())


@pytest.mark.parametrize("T,K,N,parts,tile_n", [(1000, 8960, 1536, 2, 0), (77, 192, 328, 1, 128), (640, 1536, 1536, 1, 256),
                                                 (640, 1536, 1536, 1, 512), (4096, 3584, 3584, 1, 512), (4096, 3584, 3584, 2, 256)])
def test_gemm_residual(T, K, N, parts, tile_n):
    from paper_2605_11581_b200 import prefill as P

    g = torch.Generator(device="cuda").manual_seed(T + K)
    x = torch.randn(T, K, device="cuda", generator=g)
    w = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    out = torch.randn(T, N, device="cuda", generator=g)
    xp = _planes(x, parts)
    want = out.double() + xp.double().sum(0) @ w.double().T
    P.gemm(xp, w, out, epilogue=P.EPI_RESID, tile_n=tile_n)
    err = (out.double() - want).abs().max().item()
    assert err <= 4e-5 * max(1.0, want.abs().max().item()), err


@pytest.mark.parametrize("T,K,I,parts,tile_n", [(520, 1536, 1280, 2, 256), (130, 512, 512, 1, 128), (33, 64, 704, 2, 256),
                                                 (520, 1536, 1280, 2, 512), (33, 64, 704, 1, 512), (2500, 256, 9600, 1, 512)])
def test_gemm_swiglu(T, K, I, parts, tile_n):
    """Fused gate/up GEMM: silu(gate) * up, split into bf16 planes, on an interleaved (and zero-padded) weight."""
    from paper_2605_11581_b200 import prefill as P

    g = torch.Generator(device="cuda").manual_seed(T + I)
    x = torch.randn(T, K, device="cuda", generator=g)
    wg = (torch.randn(I, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    wu = (torch.randn(I, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    w = P.interleave_gate_up(wg, wu, block=64 if tile_n == 128 else 128)
    i_pad = w.shape[0] // 2
    xp = _planes(x, parts)
    xs = xp.double().sum(0)
    want = torch.nn.functional.silu(xs @ wg.double().T) * (xs @ wu.double().T)
    out = torch.full((parts, T, i_pad), float("nan"), dtype=torch.bfloat16, device="cuda")
    P.gemm(xp, w, out, epilogue=P.EPI_SWIGLU, tile_n=tile_n)
    got = out.double().sum(0)
    assert got[:, I:].abs().max().item() == 0 if i_pad > I else True
    tol = (2e-4 if parts == 2 else 8e-3) * max(1.0, want.abs().max().item())
    assert (got[:, :I] - want).abs().max().item() <= tol


def test_gemm_rejects_bad_arguments():
    from paper_2605_11581_b200 import prefill as P
    from paper_2605_11581_b200.plugin import AdamkError

    x = torch.zeros(1, 16, 60, dtype=torch.bfloat16, device="cuda")   # K not a multiple of 8
    w = torch.zeros(16, 60, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(AdamkError):
        P.gemm(x, w, torch.zeros(16, 16, device="cuda"))
    with pytest.raises(AdamkError):
        P.gemm(torch.zeros(1, 16, 64, dtype=torch.bfloat16), torch.zeros(16, 64, dtype=torch.bfloat16), torch.zeros(16, 16))


@pytest.mark.parametrize("cfg,planes", [(TINY, 2), (TINY_QWEN3, 2), (D128, 2), (D128_Q3, 2), (D128, 1), (D128_Q3, 1)])
def test_prefill_fills_the_cache_like_the_oracle(cfg, planes):
    from oracle.decode_ref import RefDecoder, _rmsnorm
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.prefill import TensorCorePrefill
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights, rope_table

    T, max_ctx = 150, 256
    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, max_ctx)
    ref = RefDecoder(cfg, w, max_ctx, cos, sin)
    g = torch.Generator().manual_seed(3)
    prompt = torch.randint(0, cfg.vocab, (T,), generator=g)
    want_logits = ref.prefill(prompt.tolist())
    plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=max_ctx)
    plug.bind_weights(w)
    pre = TensorCorePrefill(cfg, w, plug, planes=planes)
    h = pre.run(prompt.cuda())
    torch.cuda.synchronize()
    kc, vc = plug.kv_view()
    for got, want in ((kc, ref.k_cache), (vc, ref.v_cache)):
        a = got[:, 0, :, :T].float().cpu().numpy()
        b = want[:, 0, :, :T].float().numpy()
        if planes == 2:
            # layer 0 does not depend on attention: one bf16 ulp, almost all bit-identical.  Deeper layers see the flash
            # kernel's bf16 P (2^-9 relative): up to two bf16 ulps on a per-cent of the entries
            np.testing.assert_allclose(a[0], b[0], atol=5e-3, rtol=8e-3)
            np.testing.assert_allclose(a, b, atol=2e-2, rtol=1.6e-2)
            assert (a[0] == b[0]).mean() > 0.99 and (a == b).mean() > 0.6, ((a[0] == b[0]).mean(), (a == b).mean())
        else:
            np.testing.assert_allclose(a, b, atol=6e-2, rtol=5e-2)
    hn = _rmsnorm(h[-1:].cpu(), ref.final_norm, cfg.rms_eps)
    logits = (hn @ ref.lm_head.T)[0]
    diff = (logits - want_logits).abs().max().item()
    print(f"prefill {cfg.name} planes {planes}: max |logit diff| of the last position {diff:.2e}")
    assert diff <= (2e-2 if planes == 2 else 2e-1), diff      # north-star bound with fp32-accurate GEMMs and bf16 flash attention
    assert pre.launches == 1 + cfg.n_layers * 9   # own kernels only: embed + per layer 2 norms, 4 GEMMs, rope/cache, V^T, flash attention
    plug.close()


def test_chunked_prefill_extends_the_cache():
    """Two chunks (pos0 = 0, then pos0 = 96) give the cache of one pass."""
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.prefill import TensorCorePrefill
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights

    cfg = D128
    w = random_weights(cfg, seed=1)
    g = torch.Generator().manual_seed(5)
    prompt = torch.randint(0, cfg.vocab, (160,), generator=g).cuda()
    caches = []
    for chunks in ((160,), (96, 64)):
        plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=256)
        plug.bind_weights(w)
        pre = TensorCorePrefill(cfg, w, plug, planes=2)
        pos = 0
        for n in chunks:
            pre.run(prompt[pos:pos + n], pos0=pos)
            pos += n
        torch.cuda.synchronize()
        kc, vc = plug.kv_view()
        caches.append((kc[:, 0, :, :160].float().cpu(), vc[:, 0, :, :160].float().cpu()))
        plug.close()
    for a, b in zip(*caches):
        assert (a == b).float().mean() > 0.8
        np.testing.assert_allclose(a.numpy(), b.numpy(), atol=5e-3, rtol=8e-3)


@pytest.mark.parametrize("cfg", [D128_Q3, TINY])
def test_hybrid_engine_tensor_prefill_matches_oracle(cfg):
    """PAPER.md:244-249 end to end on hand-written kernels: tensor-core Prefill fills the cache, the first generated
    token already comes from a MegaKernel launch, the greedy continuation is the oracle's."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.engine import HybridEngine
    from paper_2605_11581_b200.schedules import default_schedule
    from paper_2605_11581_b200.weights import random_weights, rope_table

    w = random_weights(cfg, seed=0)
    cos, sin = rope_table(cfg, 256)
    ref = RefDecoder(cfg, w, 256, cos, sin)
    g = torch.Generator().manual_seed(7)
    prompt = torch.randint(0, cfg.vocab, (150,), generator=g).tolist()
    want, logits = ref.generate(prompt, 24)
    eng = HybridEngine(cfg, w, max_ctx=256, schedule=default_schedule(cfg), prefill_backend="tensor", prefill_planes=2)
    res = eng.generate(prompt, 24)
    srt = torch.stack(logits).sort(dim=1).values
    margin = (srt[:, -1] - srt[:, -2]).numpy()
    first_tie = int(np.argmax(margin < 1e-3)) if (margin < 1e-3).any() else 24
    assert res.tokens[:first_tie] == want[:first_tie] and first_tie >= 12
    assert res.prefill_launches == 0 and res.decode_launches == 24
    eng.close()


@pytest.mark.parametrize("D,nq,nkv,T,pos0,qscale", [(128, 4, 2, 300, 0, 1), (128, 12, 2, 1000, 0, 1), (64, 4, 2, 130, 0, 1), (64, 2, 1, 1, 0, 1),
                                                      (128, 8, 8, 128, 0, 1), (128, 6, 1, 200, 96, 1), (64, 4, 4, 257, 300, 1),
                                                      (128, 28, 4, 4096, 0, 1), (128, 4, 2, 1500, 0, 12), (64, 4, 2, 900, 70, 12),
                                                      (128, 2, 1, 2048, 0, 40)])
def test_flash_attention_matches_fp32_reference(D, nq, nkv, T, pos0, qscale):
    _flash_case(D, nq, nkv, T, pos0, qscale)


@pytest.mark.parametrize("D,nq,nkv,T,pos0,qscale", [(128, 4, 2, 700, 0, 1), (64, 4, 2, 300, 70, 12), (128, 2, 1, 1024, 0, 40)])
def test_flash_attention_one_tile_kernel_on_long_passes(D, nq, nkv, T, pos0, qscale):
    """`adamk_prefill_attention_set_kernel(1)`: the one-tile kernel (two softmax warpgroups per q row) is what short passes
    use; forced onto longer ones it must agree with the same reference (ring wrap-around, lazy rescale)."""
    from paper_2605_11581_b200.prefill import _lib

    lib = _lib()
    lib.adamk_prefill_attention_set_kernel(1)
    try:
        _flash_case(D, nq, nkv, T, pos0, qscale)
    finally:
        lib.adamk_prefill_attention_set_kernel(0)


def _flash_case(D, nq, nkv, T, pos0, qscale):
    """csrc/prefill_attn.cu (tcgen05 QK^T and PV, softmax out of tensor memory) against a plain fp32 causal attention on
    the same bf16 q / k / v: GQA group sizes 1-7, ragged last tiles, a single row, chunked prefill (pos0 > 0), the
    Qwen2.5-7B shape at 4096 tokens.  ``qscale`` > 1 sharpens the scores (maxima that keep growing by many powers of two
    from block to block), which is what drives the kernel's lazy rescale of the output in tensor memory.  Tolerance: P
    and the output planes are bf16 (2^-9 relative)."""
    from paper_2605_11581_b200.prefill import _attn_ok, _lib, _ptr, _stream

    lib = _lib()
    g = torch.Generator(device="cuda").manual_seed(D + T + pos0)
    ctx, max_ctx = pos0 + T, pos0 + T + 37
    ctx_pad = -(-ctx // 64) * 64
    q = (qscale * torch.randn(nq, T, D, device="cuda", generator=g)).to(torch.bfloat16)
    k = torch.randn(nkv, max_ctx, D, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(nkv, max_ctx, D, device="cuda", generator=g).to(torch.bfloat16)
    k[:, ctx:] = float("nan")                       # rows past the context must never reach the output
    v[:, ctx:] = float("nan")
    vt = torch.full((nkv, D, ctx_pad), float("nan"), device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(2, T, nq * D, device="cuda", dtype=torch.bfloat16)
    _attn_ok(lib.adamk_prefill_vt(_ptr(v), nkv, D, max_ctx, ctx, ctx_pad, _ptr(vt), _stream()))
    _attn_ok(lib.adamk_prefill_attention(_ptr(q), _ptr(k), _ptr(vt), T, pos0, nq, nkv, D, max_ctx, ctx_pad, _ptr(out), 2, _stream()))
    torch.cuda.synchronize()
    assert torch.equal(vt[:, :, :ctx], v[:, :ctx].transpose(1, 2)) and (vt[:, :, ctx:] == 0).all()
    G = nq // nkv
    qf, kf, vf = q.float(), k[:, :ctx].float().repeat_interleave(G, 0), v[:, :ctx].float().repeat_interleave(G, 0)
    s = torch.einsum("htd,hcd->htc", qf, kf) / D ** 0.5
    mask = torch.arange(ctx, device="cuda")[None, :] > (pos0 + torch.arange(T, device="cuda"))[:, None]
    s.masked_fill_(mask[None], float("-inf"))
    want = torch.einsum("htc,hcd->htd", torch.softmax(s, dim=-1), vf).transpose(0, 1).reshape(T, nq * D)
    got = out[0].float() + out[1].float()
    assert torch.isfinite(got).all()
    err = (got - want).abs().max().item()
    assert err <= 2e-2, err
    assert (got - want).abs().mean().item() <= 1.5e-3
    # one plane = the bf16 rounding of the two-plane value
    assert (out[0].float() - got).abs().max().item() <= 2 ** -8 * got.abs().max().item()
