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

PREFILL_EXPORTS = ("adamk_prefill_last_error", "adamk_prefill_set_pdl", "adamk_prefill_set_plane_quarters", "adamk_prefill_set_walk", "adamk_prefill_set_trace", "adamk_prefill_prefetch_next",
                   "adamk_prefill_gemm_plan", "adamk_prefill_gemm", "adamk_prefill_embed", "adamk_prefill_rmsnorm_split",
                   "adamk_prefill_split", "adamk_prefill_rope_store", "adamk_batch_rope_store", "adamk_batch_attention_workspace",
                   "adamk_batch_attention", "adamk_batch_argmax", "adamk_batch_argmax_sliced", "adamk_batch_argmax_workspace", "adamk_batch_swiglu_split", "adamk_batch_rmsnorm_split", "adamk_batch_embed",
                   "adamk_prefill_attention", "adamk_prefill_vt", "adamk_prefill_attention_last_error", "adamk_prefill_attention_set_kernel",
                   "adamk_prefill", "adamk_prefill_workspace_bytes", "adamk_prefill_pass_last_error")


class _PassModel(C.Structure):          # include/adamk_prefill.h: AdamkPrefillModel
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("n_q_heads", C.c_int), ("n_kv_heads", C.c_int), ("head_dim", C.c_int),
                ("intermediate_padded", C.c_int), ("max_ctx", C.c_int), ("rms_eps", C.c_float), ("kv_layer_stride", C.c_longlong)]


_PASS_LAYER_FIELDS = ("ln1", "ln2", "wqkv", "bqkv", "wo", "wgu", "wdown", "q_norm", "k_norm")


class _PassLayer(C.Structure):          # include/adamk_prefill.h: AdamkPrefillLayer
    _fields_ = [(n, C.c_void_p) for n in _PASS_LAYER_FIELDS]

_declared = False


def _lib():
    global _declared
    lib = load_library()
    if not _declared:
        vp, i, ll, f = C.c_void_p, C.c_int, C.c_longlong, C.c_float
        lib.adamk_prefill_last_error.restype = C.c_char_p
        lib.adamk_prefill_set_pdl.argtypes = [i]
        lib.adamk_prefill_set_pdl.restype = None
        lib.adamk_prefill_set_plane_quarters.argtypes = [i]
        lib.adamk_prefill_set_plane_quarters.restype = None
        lib.adamk_prefill_set_walk.argtypes = [i]
        lib.adamk_prefill_set_walk.restype = None
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
        lib.adamk_prefill_attention_set_kernel.argtypes = [i]
        lib.adamk_prefill_attention_set_kernel.restype = None
        lib.adamk_prefill_pass_last_error.restype = C.c_char_p
        lib.adamk_prefill_workspace_bytes.argtypes = [C.POINTER(_PassModel), i, i, i]
        lib.adamk_prefill_workspace_bytes.restype = C.c_size_t
        lib.adamk_prefill.argtypes = [C.POINTER(_PassModel), C.POINTER(_PassLayer), vp, vp, vp, vp, i, i, i, vp, vp, vp, vp, vp]
        lib.adamk_prefill_rmsnorm_split.argtypes = [vp, vp, f, i, i, vp, i, vp]
        lib.adamk_prefill_split.argtypes = [vp, ll, vp, i, vp]
        lib.adamk_prefill_rope_store.argtypes = [vp, i, i, i, i, vp, vp, f, vp, vp, i, i, vp, i, vp, vp, vp]
        lib.adamk_batch_rope_store.argtypes = [vp, i, i, i, i, vp, vp, f, vp, vp, vp, ll, i, vp, vp, vp, vp]
        lib.adamk_batch_attention_workspace.argtypes = [i, i, i, i]
        lib.adamk_batch_attention_workspace.restype = C.c_size_t
        lib.adamk_batch_attention.argtypes = [vp, vp, vp, vp, i, i, i, i, i, ll, vp, vp, i, vp]
        lib.adamk_batch_argmax.argtypes = [vp, i, i, vp, vp, vp, vp]
        lib.adamk_batch_argmax_sliced.argtypes = [vp, i, i, vp, vp, vp, vp, vp]
        lib.adamk_batch_argmax_workspace.argtypes = [i]
        lib.adamk_batch_argmax_workspace.restype = C.c_size_t
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
        self._ws, self._pass = None, None
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
        cfg, plug, P, lib = self.cfg, self.plugin, self.planes, _lib()
        T = int(toks.numel())
        if T == 0:
            return torch.empty(0, cfg.hidden, device=plug.device)
        if pos0 + T > plug.max_ctx:
            raise ValueError("prompt does not fit the KV cache")
        dev = plug.device
        toks32 = toks.to(device=dev, dtype=torch.int32).contiguous()
        model, layers = self._pass_args()
        need = lib.adamk_prefill_workspace_bytes(C.byref(model), T, pos0, P)
        if need == 0:
            raise AdamkError(-1, "adamk_prefill_workspace_bytes rejected the model / shape")
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=dev)
        h = torch.empty(T, cfg.hidden, dtype=torch.float32, device=dev)
        cos, sin = plug._rope
        kc, vc = plug.kv_view()
        # ONE library call enqueues the whole pass (csrc/prefill_pass.cu): 1 + 9 launches per layer
        if lib.adamk_prefill(C.byref(model), layers, _ptr(self.embed), _ptr(cos), _ptr(sin), _ptr(toks32), T, pos0, P,
                             _ptr(kc[0, 0]), _ptr(vc[0, 0]), _ptr(self._ws), _ptr(h), _stream()) != 0:
            raise AdamkError(-1, (lib.adamk_prefill_pass_last_error() or b"").decode())
        self.launches += 1 + 9 * len(self.layers)
        return h

    def _pass_args(self):
        """The C description of the model and its prepared weights (cached; tensors stay owned by ``self.layers``)."""
        if self._pass is None:
            cfg, plug = self.cfg, self.plugin
            kc, _ = plug.kv_view()
            model = _PassModel(len(self.layers), cfg.hidden, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, self.layers[0]["i_pad"],
                               plug.max_ctx, cfg.rms_eps, kc.stride(0) * kc.element_size())
            arr = (_PassLayer * len(self.layers))()
            for i, lw in enumerate(self.layers):
                for name in _PASS_LAYER_FIELDS:
                    t = lw[name]
                    setattr(arr[i], name, None if t is None else t.data_ptr())
            self._pass = (model, arr)
        return self._pass
