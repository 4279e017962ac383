"""ctypes binding of libadamk.so: the MegaKernel plugin entry point.

The reference describes this layer only in prose (``PAPER.md:244-249``: the
MegaKernel is embedded "via a Plugin mechanism", Decode switches to it); see
include/adamk.h for the C ABI and INTEGRATION.md for the binding a reference
maintainer would add.  PyTorch is used for device-buffer ownership only.

There is no CPU fallback: importing works without a GPU (so host logic can be
tested), but constructing a plugin without the built library or without a CUDA
device raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from .build import LIB
from .model_config import ModelConfig
from .task_table import KernelSchedule, TaskTable, build_task_table
from .weights import DecoderWeights, rope_table

ABI_VERSION = 2


class AdamkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"adamk error {code}: {msg}")
        self.code = code


class _ModelDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "hidden", "n_layers", "n_q_heads", "n_kv_heads", "head_dim", "intermediate", "vocab",
        "max_ctx", "max_batch", "qkv_bias", "qk_norm", "tied_embed")] + [
        ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


_LAYER_FIELDS = ("ln1", "wq", "wk", "wv", "bq", "bk", "bv", "q_norm", "k_norm", "wo", "ln2",
                 "wgate", "wup", "wdown")


class _LayerWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _LAYER_FIELDS]


_QUANT_FIELDS = tuple(f"{kind}_{name}" for name in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown") for kind in ("q", "s"))


class _W4A16Layer(C.Structure):   # include/adamk.h: AdamkW4A16Layer
    _fields_ = [(n, C.c_void_p) for n in _QUANT_FIELDS]


class _WeightPtrs(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("final_norm", C.c_void_p), ("lm_head", C.c_void_p),
                ("layers", C.POINTER(_LayerWeights)), ("rope_cos", C.c_void_p), ("rope_sin", C.c_void_p)]


EXPORTS = (
    "adamk_abi_version", "adamk_device_sm_count", "adamk_last_error", "adamk_create", "adamk_destroy",
    "adamk_packed_bytes", "adamk_bind_weights", "adamk_bind_peers", "adamk_workspace_bytes",
    "adamk_workspace_init", "adamk_kv_cache_bytes", "adamk_decode_step", "adamk_device_status",
    "adamk_stream_probe", "adamk_trace_bytes", "adamk_set_trace", "adamk_share_weights", "adamk_bind_weights_w4a16",
    "adamk_decode_step_host",
)

_lib = None


def load_library() -> C.CDLL:
    """dlopen libadamk.so (built in-tree by ``build.py``) and declare prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    import os
    from pathlib import Path

    path = Path(os.environ.get("ADAMK_LIB", str(LIB)))   # override: A/B runs of two builds of the same ABI
    if not path.exists():
        raise AdamkError(-100, f"{path} is not built; run `python -m paper_2605_11581_b200.build` "
                               "(there is no CPU fallback for the decode path)")
    lib = C.CDLL(str(path))
    lib.adamk_abi_version.restype = C.c_int
    lib.adamk_last_error.restype = C.c_char_p
    lib.adamk_device_sm_count.argtypes = [C.c_int, C.POINTER(C.c_int)]
    lib.adamk_create.argtypes = [C.POINTER(_ModelDesc), C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                                 C.POINTER(C.c_void_p)]
    lib.adamk_destroy.argtypes = [C.c_void_p]
    lib.adamk_destroy.restype = None
    lib.adamk_set_trace.argtypes = [C.c_void_p, C.c_void_p]
    for name in ("adamk_packed_bytes", "adamk_workspace_bytes", "adamk_kv_cache_bytes", "adamk_trace_bytes"):
        getattr(lib, name).argtypes = [C.c_void_p]
        getattr(lib, name).restype = C.c_size_t
    lib.adamk_bind_weights.argtypes = [C.c_void_p, C.POINTER(_WeightPtrs), C.c_void_p, C.c_void_p]
    lib.adamk_bind_weights_w4a16.argtypes = [C.c_void_p, C.POINTER(_WeightPtrs), C.POINTER(_W4A16Layer), C.c_void_p, C.c_void_p]
    lib.adamk_bind_peers.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int]
    lib.adamk_share_weights.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_WeightPtrs)]
    lib.adamk_workspace_init.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.adamk_decode_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.adamk_decode_step_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int] + [C.c_void_p] * 9
    lib.adamk_device_status.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    lib.adamk_stream_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    if lib.adamk_abi_version() != ABI_VERSION:
        raise AdamkError(-101, "libadamk.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


def _check(lib, code: int) -> None:
    if code != 0:
        raise AdamkError(code, (lib.adamk_last_error() or b"").decode())


def device_sm_count(device: int = 0) -> int:
    lib = load_library()
    n = C.c_int(0)
    _check(lib, lib.adamk_device_sm_count(device, C.byref(n)))
    return n.value


@dataclass
class StepOutput:
    next_token: torch.Tensor            # int32 [batch] (device)
    logits: torch.Tensor | None         # fp32 [batch, vocab] (device) or None


class MegaKernelPlugin:
    """One decode MegaKernel instance bound to one GPU.

    ``schedule`` carries the solidified pipeline parameters (from
    ``KernelSchedule.from_plan(solidified_trace.plan)``); the whole-model task
    table is derived from it and the model config at construction."""

    def __init__(self, cfg: ModelConfig, schedule: KernelSchedule, max_ctx: int, device: int | str = 0,
                 n_sms: int | None = None, tp_rank: int = 0, tp_size: int = 1):
        """``cfg`` holds the dimensions of THIS rank (``full_cfg.shard(tp_size)``); with ``tp_size > 1`` call
        :meth:`bind_peers` with every rank's workspace before the first step."""
        if not torch.cuda.is_available():
            raise AdamkError(-102, "no CUDA device: the decode MegaKernel has no CPU fallback")
        self.lib = load_library()
        self.cfg, self.schedule, self.max_ctx = cfg, schedule, int(max_ctx)
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        torch.cuda.set_device(self.device)
        self.n_sms = n_sms or device_sm_count(self.device.index or 0)
        self.table: TaskTable = build_task_table(cfg, schedule, n_sms=self.n_sms, batch=1)
        desc = _ModelDesc(cfg.hidden, cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim,
                          cfg.intermediate, cfg.vocab, self.max_ctx, 1, int(cfg.qkv_bias), int(cfg.qk_norm),
                          int(cfg.tied_embed), cfg.rms_eps, cfg.rope_theta)
        blob = self.table.blob
        self._blob = C.create_string_buffer(blob, len(blob))
        h = C.c_void_p()
        self.tp_rank, self.tp_size = int(tp_rank), int(tp_size)
        _check(self.lib, self.lib.adamk_create(C.byref(desc), self._blob, len(blob), self.tp_rank, self.tp_size, C.byref(h)))
        self._h = h
        self._weights: DecoderWeights | None = None
        self.packed: torch.Tensor | None = None
        self.workspace = torch.empty(self.lib.adamk_workspace_bytes(h), dtype=torch.uint8, device=self.device)
        self._stream_ptr = lambda: C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(self.lib, self.lib.adamk_workspace_init(h, C.c_void_p(self.workspace.data_ptr()), self._stream_ptr()))
        kv_elems = self.lib.adamk_kv_cache_bytes(h) // 2
        self.k_cache = torch.zeros(kv_elems, dtype=torch.bfloat16, device=self.device)
        self.v_cache = torch.zeros(kv_elems, dtype=torch.bfloat16, device=self.device)
        self._state = torch.zeros(2, dtype=torch.int32, device=self.device)   # token | position, adjacent: one H2D copy
        self.tokens = self._state[0:1]
        self.positions = self._state[1:2]
        self._host_io = None                      # pinned int32[3]: token, position | next token (decode_step_host)
        self.next_token = torch.zeros(1, dtype=torch.int32, device=self.device)
        # logits of the whole vocabulary; a tensor-parallel rank fills its own slice [rank * V/tp, (rank + 1) * V/tp)
        self.logits = torch.zeros(1, cfg.vocab * self.tp_size, dtype=torch.float32, device=self.device)
        self.launches = 0

    @classmethod
    def from_trace(cls, cfg: ModelConfig, trace_text, max_ctx: int, device: int | str = 0, graph_text: str | None = None,
                   hw_text: str | None = None, **kernel_knobs):
        """Build the plugin from a SolidifiedTrace (``mkplan search --out``; reference ``search.py:79-171``).
        ``KernelSchedule.from_plan`` lowers the plan: tile -> ring stage geometry, consumer warps, ``stride_eff`` -> the
        Loader's stages in flight, ``n_stage`` / ``window`` checked against the ring depth Eq.1 / Eq.2 give on this
        kernel's shared-memory accounting.  With the trace's ``graph_text`` / ``hw_text`` the plan's Loader / Consumer
        programs are checked against the order the kernel replays (``solidify.check_program_order``).  Run-time knobs
        the planner does not model (split-KV chunk, L2 prefetch window, fused down projection) come as ``kernel_knobs``."""
        from .mkplan.search import parse_trace
        from .solidify import check_program_order, schedule_from_trace

        trace = parse_trace(trace_text if isinstance(trace_text, (bytes, bytearray)) else str(trace_text).encode())
        if graph_text is not None and hw_text is not None:
            check_program_order(trace, graph_text, hw_text)
        n_sms = device_sm_count(device if isinstance(device, int) else torch.device(device).index or 0)
        return cls(cfg, schedule_from_trace(cfg, trace, kernel_knobs, n_sms=n_sms), max_ctx, device=device)

    # -- weights -------------------------------------------------------------
    def bind_weights(self, w, keep_source: bool = False) -> None:
        """Repack the weights into the per-SM tile-major streams: HF-layout bf16 ``DecoderWeights``, or -- for a
        schedule with ``w4a16`` -- ``quant.QuantizedWeights`` (4-bit codes + fp16 group scales of the layer projections;
        embedding, norms, biases and LM head come from its bf16 ``base``)."""
        cfg = self.cfg
        quantized = hasattr(w, "base")
        if quantized != bool(self.schedule.w4a16):
            raise AdamkError(-101, "a w4a16 schedule takes quant.QuantizedWeights, a bf16 schedule DecoderWeights")
        qw = w.to(self.device) if quantized else None
        w = qw.base if quantized else w.to(self.device)
        cos, sin = rope_table(cfg, self.max_ctx)
        self._rope = (cos.to(self.device), sin.to(self.device))
        layers = (_LayerWeights * cfg.n_layers)()
        for i, lw in enumerate(w.layers):
            for name in _LAYER_FIELDS:
                t = getattr(lw, name)
                if t is not None:
                    assert t.dtype == torch.bfloat16 and t.is_contiguous()
                setattr(layers[i], name, None if t is None else t.data_ptr())
        ptrs = _WeightPtrs(w.embed.data_ptr(), w.final_norm.data_ptr(),
                           None if w.lm_head is None else w.lm_head.data_ptr(),
                           layers, self._rope[0].data_ptr(), self._rope[1].data_ptr())
        self.packed = torch.empty(self.lib.adamk_packed_bytes(self._h), dtype=torch.uint8, device=self.device)
        if quantized:
            qlayers = (_W4A16Layer * cfg.n_layers)()
            for i, ql in enumerate(qw.layers):
                for name, m in ql.items():
                    assert m.q.dtype == torch.uint8 and m.s.dtype == torch.float16 and m.q.is_contiguous() and m.s.is_contiguous()
                    setattr(qlayers[i], f"q_{name}", m.q.data_ptr())
                    setattr(qlayers[i], f"s_{name}", m.s.data_ptr())
            _check(self.lib, self.lib.adamk_bind_weights_w4a16(self._h, C.byref(ptrs), qlayers, C.c_void_p(self.packed.data_ptr()),
                                                               self._stream_ptr()))
        else:
            _check(self.lib, self.lib.adamk_bind_weights(self._h, C.byref(ptrs), C.c_void_p(self.packed.data_ptr()),
                                                         self._stream_ptr()))
        self._embed = w.embed                      # the kernel gathers embedding rows from the source table
        self._weights = (qw if quantized else w) if keep_source else None

    def share_weights(self, owner: "MegaKernelPlugin") -> None:
        """Stream the packed weights ``owner`` has bound (identical task table required) instead of repacking."""
        assert owner.packed is not None
        self._rope = owner._rope
        ptrs = _WeightPtrs(owner._embed.data_ptr(), None, None, None, self._rope[0].data_ptr(), self._rope[1].data_ptr())
        _check(self.lib, self.lib.adamk_share_weights(self._h, owner._h, C.byref(ptrs)))
        self.packed, self._embed = owner.packed, owner._embed

    def bind_peers(self, peer_workspaces) -> None:
        """Tensor parallelism: device pointers (or tensors) of EVERY rank's workspace, own rank included, in rank
        order.  On one node these are peer-mapped allocations (CUDA IPC / cuMem handles exchanged once through
        ``torch.distributed``, see dist_utils.share_workspaces); the kernel stores its partial rows into them."""
        ptrs = [int(w.data_ptr()) if hasattr(w, "data_ptr") else int(w) for w in peer_workspaces]
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        _check(self.lib, self.lib.adamk_bind_peers(self._h, arr, len(ptrs)))
        self._peers = list(peer_workspaces)   # keep the mappings alive

    # -- decode ----------------------------------------------------------------
    def set_state(self, token: int, position: int) -> None:
        self.tokens.fill_(int(token))
        self.positions.fill_(int(position))

    def enqueue(self, want_logits: bool = False, auto_advance: bool = True) -> None:
        """Enqueue ONE decode step (one kernel launch) on the current stream using
        the device-resident token/position state."""
        _check(self.lib, self.lib.adamk_decode_step(
            self._h, C.c_void_p(self.tokens.data_ptr()), C.c_void_p(self.positions.data_ptr()), 1,
            C.c_void_p(self.k_cache.data_ptr()), C.c_void_p(self.v_cache.data_ptr()),
            C.c_void_p(self.workspace.data_ptr()),
            C.c_void_p(self.logits.data_ptr()) if want_logits else None,
            C.c_void_p(self.next_token.data_ptr()), int(auto_advance), self._stream_ptr()))
        self.launches += 1

    def decode_step(self, token: int, position: int, want_logits: bool = True) -> StepOutput:
        """Host-facing step: host token/position in, device outputs out (no sync)."""
        self.set_state(token, position)
        self.enqueue(want_logits=want_logits, auto_advance=False)
        return StepOutput(self.next_token, self.logits if want_logits else None)

    def decode_step_host(self, token: int, position: int, want_logits: bool = False) -> int:
        """The serving engine's per-token hook with HOST buffers (``adamk_decode_step_host``): token and position go
        from pinned host memory to the device, one launch, the greedy next token comes back; returns it."""
        if self._host_io is None:
            self._host_io = torch.zeros(3, dtype=torch.int32).pin_memory()
            self._host_np = self._host_io.numpy()
            self._host_args = {}
        io = self._host_np
        io[0], io[1] = token, position
        stream = torch.cuda.current_stream(self.device).cuda_stream
        key = (bool(want_logits), stream)
        args = self._host_args.get(key)
        if args is None:        # every argument but the token and the position is fixed: converted once per (logits, stream)
            base = self._host_io.data_ptr()
            args = (self._h, C.c_void_p(base), C.c_void_p(base + 4), 1,
                    C.c_void_p(self.tokens.data_ptr()), C.c_void_p(self.positions.data_ptr()),
                    C.c_void_p(self.k_cache.data_ptr()), C.c_void_p(self.v_cache.data_ptr()),
                    C.c_void_p(self.workspace.data_ptr()),
                    C.c_void_p(self.logits.data_ptr()) if want_logits else None,
                    C.c_void_p(self.next_token.data_ptr()), C.c_void_p(base + 8), C.c_void_p(stream))
            self._host_args[key] = args
        _check(self.lib, self.lib.adamk_decode_step_host(*args))
        self.launches += 1
        return int(io[2])

    def check(self) -> None:
        """Synchronise and raise if the kernel reported an error."""
        try:
            torch.cuda.synchronize(self.device)
        finally:
            info = (C.c_int32 * 8)()
            code = self.lib.adamk_device_status(self._h, info)
            if code != 0:
                raise AdamkError(-5, f"device error {code}: sm={info[1]} task={info[2]} a={info[3]} "
                                     f"b={info[4]} c={info[5]} tid={info[6]}")

    def stream_probe(self, mode: int = 1) -> None:
        if not hasattr(self, "_sink"):
            self._sink = torch.zeros(self.n_sms * 64, dtype=torch.float32, device=self.device)
        _check(self.lib, self.lib.adamk_stream_probe(self._h, C.c_void_p(self._sink.data_ptr()), mode,
                                                     self._stream_ptr()))

    def enable_trace(self, on: bool = True) -> torch.Tensor | None:
        """Per-task %globaltimer stamps [n_tasks, 8] (0 start, 1 dependency met, 2 prologue done, 7 end)."""
        if on:
            n = self.lib.adamk_trace_bytes(self._h) // 8
            self.trace = torch.zeros(n // 8, 8, dtype=torch.int64, device=self.device)
            _check(self.lib, self.lib.adamk_set_trace(self._h, C.c_void_p(self.trace.data_ptr())))
            return self.trace
        _check(self.lib, self.lib.adamk_set_trace(self._h, None))
        self.trace = None
        return None

    def kv_view(self) -> tuple[torch.Tensor, torch.Tensor]:
        cfg = self.cfg
        shape = (cfg.n_layers, 1, cfg.n_kv_heads, self.max_ctx, cfg.head_dim)
        return self.k_cache.view(shape), self.v_cache.view(shape)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.adamk_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class BatchLanes:
    """Batched decode by SM partitioning: ``batch`` instances of the batch-1 kernel on disjoint SM subsets
    (n_sms // batch each), one sequence per lane, all streaming ONE packed weight buffer.  The lanes start
    together and do identical work, so the second reader of a weight stage finds it in L2 and HBM still sees
    each weight once per step; correctness is that of the batch-1 kernel by construction.  (SURVEY.md 8(f).1's
    tensor-core path for batch >= 8 is a separate kernel and not built yet; this is the CUDA-core path for
    small batches.)"""

    def __init__(self, cfg: ModelConfig, schedule: KernelSchedule, max_ctx: int, batch: int, device: int = 0):
        from .schedules import fit_schedule

        total = device_sm_count(device)
        self.batch = int(batch)
        schedule = fit_schedule(cfg, schedule, n_sms=total // self.batch)   # ring depth / fused down projection for the lane's SM count
        self.lanes = [MegaKernelPlugin(cfg, schedule, max_ctx, device=device, n_sms=total // self.batch)
                      for _ in range(self.batch)]
        self.device = self.lanes[0].device
        self.streams = [torch.cuda.Stream(self.device) for _ in range(self.batch)]
        self._fork = torch.cuda.Event()
        self._joins = [torch.cuda.Event() for _ in range(self.batch)]

    def bind_weights(self, w: DecoderWeights) -> None:
        self.lanes[0].bind_weights(w)
        for lane in self.lanes[1:]:
            lane.share_weights(self.lanes[0])

    def set_state(self, tokens, positions) -> None:
        for lane, t, p in zip(self.lanes, tokens, positions):
            lane.set_state(int(t), int(p))

    def enqueue(self, want_logits: bool = False, auto_advance: bool = True) -> None:
        """One decode step of every sequence: the lanes' kernels run concurrently, forked from and joined
        back into the current stream."""
        cur = torch.cuda.current_stream(self.device)
        self._fork.record(cur)
        for lane, st, ev in zip(self.lanes, self.streams, self._joins):
            st.wait_event(self._fork)
            with torch.cuda.stream(st):
                lane.enqueue(want_logits=want_logits, auto_advance=auto_advance)
                ev.record(st)
        for ev in self._joins:
            cur.wait_event(ev)

    def decode_step(self, tokens, positions, want_logits: bool = True) -> StepOutput:
        self.set_state(tokens, positions)
        self.enqueue(want_logits=want_logits, auto_advance=False)
        nxt = torch.cat([lane.next_token for lane in self.lanes])
        logits = torch.cat([lane.logits for lane in self.lanes]) if want_logits else None
        return StepOutput(nxt, logits)

    def check(self) -> None:
        for lane in self.lanes:
            lane.check()

    @property
    def launches(self) -> int:
        return sum(lane.launches for lane in self.lanes)

    def close(self) -> None:
        for lane in self.lanes:
            lane.close()
