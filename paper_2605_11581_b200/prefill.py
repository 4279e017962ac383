"""Prefill phase on hand-written tensor-core operators.

``PAPER.md:244-249`` runs Prefill on the serving engine's operators and Decode on the MegaKernel.  This module is
that Prefill half built from ``include/adamk_prefill.h``: a tcgen05 / tensor-memory GEMM
(``csrc/prefill_gemm.cu``) with fused bias, residual and SwiGLU epilogues, a tcgen05 causal flash-attention kernel
(``csrc/prefill_attn.cu``) and the row kernels around them (``csrc/prefill_ops.cu``).  Layer dataflow for ``T`` prompt tokens::

    h fp32 [T, H] --rmsnorm_split--> planes --GEMM(wqkv)+bias--> qkv fp32 --rope_store--> q, KV cache (bf16)
      --V^T, flash attention--> a planes --GEMM(wo) += h--> h --rmsnorm_split--> planes --GEMM(gate|up) SwiGLU--> act planes
      --GEMM(wdown) += h--> h

``planes`` = 2 keeps the decode kernel's numerical contract (fp32 activations against exact bf16 weights: each fp32
value enters the tensor cores as hi + lo bf16 planes); ``planes`` = 1 is plain bf16 activations at half the
tensor work.  Causal attention over the bf16 cache (as the decode kernel will see it) is the flash kernel in either
mode: bf16 Q / K / V / P, fp32 scores, softmax state and output -- no library operator is left on this path.  There
is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import torch

from .model_config import ModelConfig
from .plugin import AdamkError, load_library
from .weights import DecoderWeights

EPI_STORE, EPI_RESID, EPI_SWIGLU, EPI_ATOMIC = 0, 1, 2, 3
TILE_AUTO, TILE_128, TILE_256, TILE_PAIR = 0, 128, 256, 512   # include/adamk_prefill.h ADAMK_PF_TILE_*
PREFETCH_MAX_BYTES = 64 << 20   # L2 prefetch hint cap (half of the 126 MB L2)
GU_BLOCK = 128   # features per gate / up block of the interleaved weight = half of a 256-wide GEMM tile

PREFILL_EXPORTS = ("adamk_prefill_last_error", "adamk_prefill_set_pdl", "adamk_prefill_set_trace", "adamk_prefill_prefetch_next",
                   "adamk_prefill_gemm_plan", "adamk_prefill_gemm", "adamk_prefill_embed", "adamk_prefill_rmsnorm_split",
                   "adamk_prefill_split", "adamk_prefill_rope_store", "adamk_batch_rope_store", "adamk_batch_attention_workspace",
                   "adamk_batch_attention", "adamk_batch_argmax", "adamk_batch_swiglu_split", "adamk_batch_rmsnorm_split", "adamk_batch_embed",
                   "adamk_prefill_attention", "adamk_prefill_vt", "adamk_prefill_attention_last_error")

_declared = False


def _lib():
    global _declared
    lib = load_library()
    if not _declared:
        vp, i, ll, f = C.c_void_p, C.c_int, C.c_longlong, C.c_float
        lib.adamk_prefill_last_error.restype = C.c_char_p
        lib.adamk_prefill_set_pdl.argtypes = [i]
        lib.adamk_prefill_set_pdl.restype = None
        lib.adamk_prefill_set_trace.argtypes = [vp]
        lib.adamk_prefill_prefetch_next.argtypes = [vp, ll]
        lib.adamk_prefill_prefetch_next.restype = None
        lib.adamk_prefill_set_trace.restype = None
        lib.adamk_prefill_gemm.argtypes = [vp, i, i, i, vp, i, vp, vp, i, i, i, ll, i, vp]
        lib.adamk_prefill_gemm_plan.argtypes = [i, i, i, i, i, i, i, C.POINTER(C.c_int32)]
        lib.adamk_prefill_embed.argtypes = [vp, i, vp, i, vp, vp]
        lib.adamk_batch_embed.argtypes = [vp, i, vp, i, i, vp, vp]
        lib.adamk_prefill_attention.argtypes = [vp, vp, vp, i, i, i, i, i, i, i, vp, i, vp]
        lib.adamk_prefill_vt.argtypes = [vp, i, i, i, i, i, vp, vp]
        lib.adamk_prefill_attention_last_error.restype = C.c_char_p
        lib.adamk_prefill_rmsnorm_split.argtypes = [vp, vp, f, i, i, vp, i, vp]
        lib.adamk_prefill_split.argtypes = [vp, ll, vp, i, vp]
        lib.adamk_prefill_rope_store.argtypes = [vp, i, i, i, i, vp, vp, f, vp, vp, i, i, vp, i, vp, vp, vp]
        lib.adamk_batch_rope_store.argtypes = [vp, i, i, i, i, vp, vp, f, vp, vp, vp, ll, i, vp, vp, vp, vp]
        lib.adamk_batch_attention_workspace.argtypes = [i, i, i, i]
        lib.adamk_batch_attention_workspace.restype = C.c_size_t
        lib.adamk_batch_attention.argtypes = [vp, vp, vp, vp, i, i, i, i, i, ll, vp, vp, i, vp]
        lib.adamk_batch_argmax.argtypes = [vp, i, i, vp, vp, vp, vp]
        lib.adamk_batch_swiglu_split.argtypes = [vp, i, i, i, vp, i, vp]
        lib.adamk_batch_rmsnorm_split.argtypes = [vp, vp, f, i, i, vp, i, vp, ll, vp]
        _declared = True
    return lib


def _ok(code: int) -> None:
    if code != 0:
        raise AdamkError(code, (_lib().adamk_prefill_last_error() or b"").decode() or "prefill operator: invalid argument")


def _attn_ok(code: int) -> None:
    if code != 0:
        raise AdamkError(code, (_lib().adamk_prefill_attention_last_error() or b"").decode() or "prefill attention: invalid argument")


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def gemm(x_planes: torch.Tensor, w: torch.Tensor, out: torch.Tensor, bias: torch.Tensor | None = None,
         epilogue: int = EPI_STORE, tile_n: int = 0, prefetch: torch.Tensor | None = None) -> torch.Tensor:
    """``out`` (op)= sum_p x_planes[p] @ w.T on the tensor cores.  ``x_planes`` bf16 [parts, T, K], ``w`` bf16 [N, K];
    ``out`` fp32 [T, N] (STORE / RESID / ATOMIC) or bf16 [parts_out, T, N / 2] (SWIGLU, gate / up interleaved in ``w``).
    ATOMIC adds into ``out`` with fp32 atomics and lets the library split K across SMs (decode-sized T)."""
    if not x_planes.is_cuda:
        raise AdamkError(-102, "prefill operators have no CPU fallback")
    assert x_planes.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and x_planes.is_contiguous() and w.is_contiguous()
    parts, T, K = x_planes.shape
    N = w.shape[0]
    assert w.shape[1] == K and out.is_contiguous()
    if epilogue == EPI_SWIGLU:
        assert out.dtype == torch.bfloat16 and out.dim() == 3 and out.shape[1] == T and out.shape[2] == N // 2
        parts_out, ldo, stride = out.shape[0], out.shape[2], out.shape[1] * out.shape[2]
    else:
        assert out.dtype == torch.float32 and out.shape == (T, N)
        parts_out, ldo, stride = 1, N, 0
    if bias is not None:
        assert bias.dtype == torch.float32 and bias.numel() == N and epilogue in (EPI_STORE, EPI_ATOMIC)
    if prefetch is not None:       # the weight of the GEMM that follows this one: pulled into L2 by this launch's idle warps
        _lib().adamk_prefill_prefetch_next(_ptr(prefetch), min(prefetch.numel() * prefetch.element_size(), PREFETCH_MAX_BYTES))
    _ok(_lib().adamk_prefill_gemm(_ptr(x_planes), parts, T, K, _ptr(w), N, _ptr(bias), _ptr(out), ldo, epilogue, parts_out,
                                  stride, tile_n, _stream()))
    return out


PLAN_FIELDS = ("tile", "tiles", "main_items", "tail_split", "n_items", "ksplit", "kb_per_split", "stacked", "grid")


def gemm_plan(parts: int, T: int, K: int, N: int, epilogue: int = EPI_STORE, tile_n: int = 0, n_sms: int = 148) -> dict:
    """How ``gemm`` would cut this problem into work items on ``n_sms`` SMs (host arithmetic in the library; no GPU)."""
    out = (C.c_int32 * 9)()
    _ok(_lib().adamk_prefill_gemm_plan(parts, T, K, N, epilogue, tile_n, n_sms, out))
    return dict(zip(PLAN_FIELDS, out))


def interleave_gate_up(wgate: torch.Tensor, wup: torch.Tensor, block: int = GU_BLOCK) -> torch.Tensor:
    """[2 * I_pad, K]: blocks of ``block`` gate rows followed by the ``block`` up rows of the same features (zero rows
    pad I to a multiple of ``block``), so that one 2*block-wide GEMM tile holds both halves of SwiGLU."""
    I, K = wgate.shape
    I_pad = -(-I // block) * block
    g = torch.zeros(I_pad, K, dtype=wgate.dtype, device=wgate.device)
    u = torch.zeros_like(g)
    g[:I], u[:I] = wgate, wup
    return torch.stack((g.view(-1, block, K), u.view(-1, block, K)), dim=1).reshape(2 * I_pad, K).contiguous()


class TensorCorePrefill:
    """Token-parallel causal pass that fills the KV cache a ``MegaKernelPlugin`` owns."""

    def __init__(self, cfg: ModelConfig, weights: DecoderWeights, plugin, planes: int = 2, attention: str | None = None,
                 layers: list | None = None, embed: torch.Tensor | None = None):
        """``planes``: bf16 planes per fp32 activation fed to the GEMMs (1: plain bf16; 2: hi + lo, fp32-accurate).
        Attention is this library's tcgen05 flash kernel (``csrc/prefill_attn.cu``: bf16 Q / K / V / P, fp32 scores and
        output -- the flash-attention contract) for either setting; ``attention`` is accepted for compatibility with
        the first round's "bf16" / "fp32" library-operator switch and ignored.  ``layers`` / ``embed``: already prepared
        device weights (``batch_decode.BatchedDecoder`` shares its own)."""
        if planes not in (1, 2):
            raise ValueError("planes must be 1 (bf16 activations) or 2 (hi + lo, fp32-accurate)")
        if attention not in (None, "bf16", "fp32", "flash"):
            raise ValueError("attention must be 'flash' (or the legacy 'bf16' / 'fp32')")
        _lib()
        self.cfg, self.plugin, self.planes = cfg, plugin, planes
        dev = plugin.device
        self.launches = 0
        if layers is not None:
            self.embed, self.layers = embed, layers
            return
        self.embed = weights.embed.to(dev)
        self.layers = []
        for lw in weights.layers:
            wqkv = torch.cat((lw.wq, lw.wk, lw.wv), dim=0).to(dev).contiguous()
            bqkv = None
            if lw.bq is not None:
                bqkv = torch.cat((lw.bq, lw.bk, lw.bv)).to(dev).float().contiguous()
            wgu = interleave_gate_up(lw.wgate.to(dev), lw.wup.to(dev))
            i_pad = wgu.shape[0] // 2
            wdown = lw.wdown.to(dev)
            if i_pad != cfg.intermediate:
                wdown = torch.nn.functional.pad(wdown, (0, i_pad - cfg.intermediate))
            self.layers.append(dict(ln1=lw.ln1.to(dev), ln2=lw.ln2.to(dev), wqkv=wqkv, bqkv=bqkv, wo=lw.wo.to(dev).contiguous(),
                                    wgu=wgu, wdown=wdown.contiguous(), i_pad=i_pad,
                                    q_norm=None if lw.q_norm is None else lw.q_norm.to(dev),
                                    k_norm=None if lw.k_norm is None else lw.k_norm.to(dev)))
        self.launches = 0

    @torch.no_grad()
    def run(self, toks: torch.Tensor, pos0: int = 0) -> torch.Tensor:
        """Fill cache rows ``pos0 .. pos0 + T - 1`` of every layer from ``toks`` (int32 / int64 [T] on the device) and
        return the final hidden states fp32 [T, H].  ``pos0`` must be 0 unless the earlier rows are already cached
        (chunked prefill attends to them)."""
        cfg, plug, P, lib, st = self.cfg, self.plugin, self.planes, _lib(), _stream()
        T = int(toks.numel())
        if T == 0:
            return torch.empty(0, cfg.hidden, device=plug.device)
        if pos0 + T > plug.max_ctx:
            raise ValueError("prompt does not fit the KV cache")
        dev, H, D, nq, nkv = plug.device, cfg.hidden, cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
        bf = torch.bfloat16
        toks32 = toks.to(device=dev, dtype=torch.int32).contiguous()
        h = torch.empty(T, H, dtype=torch.float32, device=dev)
        xp = torch.empty(P, T, H, dtype=bf, device=dev)
        qkv = torch.empty(T, (nq + 2 * nkv) * D, dtype=torch.float32, device=dev)
        q = torch.empty(nq, T, D, dtype=bf, device=dev)
        ap = torch.empty(P, T, nq * D, dtype=bf, device=dev)
        act = torch.empty(P, T, self.layers[0]["i_pad"], dtype=bf, device=dev)
        ctx = pos0 + T
        ctx_pad = -(-ctx // 64) * 64
        vt = torch.empty(nkv, D, ctx_pad, dtype=bf, device=dev)     # V^T of the current layer (K-major operand of P.V)
        cos, sin = plug._rope
        kc, vc = plug.kv_view()
        _ok(lib.adamk_prefill_embed(_ptr(toks32), T, _ptr(self.embed), H, _ptr(h), st))
        n = 1
        for l, lw in enumerate(self.layers):
            _ok(lib.adamk_prefill_rmsnorm_split(_ptr(h), _ptr(lw["ln1"]), cfg.rms_eps, T, H, _ptr(xp), P, st))
            gemm(xp, lw["wqkv"], qkv, bias=lw["bqkv"])
            _ok(lib.adamk_prefill_rope_store(_ptr(qkv), T, nq, nkv, D, _ptr(lw["q_norm"]), _ptr(lw["k_norm"]), cfg.rms_eps,
                                             _ptr(cos), _ptr(sin), pos0, plug.max_ctx, _ptr(q), 1,
                                             _ptr(kc[l, 0]), _ptr(vc[l, 0]), st))
            # causal attention over the bf16 cache contents, as the decode kernel sees them: tcgen05 flash kernel
            _attn_ok(lib.adamk_prefill_vt(_ptr(vc[l, 0]), nkv, D, plug.max_ctx, ctx, ctx_pad, _ptr(vt), st))
            _attn_ok(lib.adamk_prefill_attention(_ptr(q), _ptr(kc[l, 0]), _ptr(vt), T, pos0, nq, nkv, D, plug.max_ctx, ctx_pad,
                                                 _ptr(ap), P, st))
            gemm(ap, lw["wo"], h, epilogue=EPI_RESID)
            _ok(lib.adamk_prefill_rmsnorm_split(_ptr(h), _ptr(lw["ln2"]), cfg.rms_eps, T, H, _ptr(xp), P, st))
            gemm(xp, lw["wgu"], act, epilogue=EPI_SWIGLU)
            gemm(act, lw["wdown"], h, epilogue=EPI_RESID)
            n += 9
        self.launches += n
        return h
