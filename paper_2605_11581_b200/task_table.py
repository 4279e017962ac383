"""Lower a solidified schedule to the static device task table.

Ada-MK's offline half ends with a ``SolidifiedTrace`` (reference
``pkg/src/mkplan/search.py:79-107``; plan fields ``tile``, ``n_stage``,
``consumer_warps``, ``stride_eff``, ``programs``, ``page_plan`` at ``:138-171``).
That artifact describes ONE SM running ONE layer's pipeline.  The online half
(paper only, ``PAPER.md:84,177-197``) replays it: Loader warps stream weight
sub-tiles into pages, Consumer warps compute, Storers publish, and "path
solidification" means no scheduling decision is left for run time.

This module is the bridge.  It maps the plan's pipeline parameters onto the
persistent sm_100a kernel's ring (``KernelSchedule``) and expands the whole
model -- every layer of every operator plus the LM head -- into a flat,
per-SM, program-ordered list of 64-byte task records with *fixed* dependency
counter targets.  The kernel (``csrc/adamk.cu``) only walks its list.

Role mapping (reference ``planner.py:60-77`` -> kernel):
  Loader   -> warp 0, one elected lane issuing ``cp.async.bulk`` (TMA) per stage
  Consumer -> warps 1..C: GEMV over the staged sub-tile, fp32 accumulate
  Storer   -> the epilogue of the consumer warps + the release of the counter
  Launcher -> the task-record fetch at the top of every task
Page states Empty/Locked/Ready (``planner.py:84-94``) are the ring slot's
``empty`` mbarrier phase / in-flight TMA / ``full`` mbarrier phase.

Stage geometry: a stage is ``rows_per_tile`` output rows by ``ktile_chunks``
256-element K chunks of bf16 = the reference's weight sub-tile
``block_n * sub_k * 2`` bytes (``graph_ir.py:308-311``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model_config import ModelConfig

MAGIC = 0x4B4D4441  # "ADMK"
VERSION = 2
HEADER_INTS = 16
TASK_INTS = 16
KCHUNK = 256           # K elements per chunk: 32 lanes x 8 bf16 (one LDS.128 per lane)
SMEM_MAX = 232448      # 227 KB opt-in shared memory per CTA on sm_100
SMEM_RESERVED = 3584   # mbarriers + reduction scratch + parameter copy ahead of the scratch/ring regions
MAX_STAGES = 16
MAX_RW = 8             # rows per consumer warp per tile (eight accumulator rows per lane)
ATTN_BLOCK = 64        # most positions per K (or V) ring stage: 8 per attention warp
ATTN_WARPS = 8         # consumer warps that take part in an attention unit
ATTN_CHUNKS_MAX = 128  # split-KV units per (sequence, kv head)
G_MAX = 8              # q heads per kv head

T_END, T_QKV, T_ATTN, T_OPROJ, T_GATEUP, T_DOWN, T_LMHEAD, T_MERGE, T_DOWNK, T_HRED = 0, 1, 2, 3, 4, 5, 6, 7, 8, 9
GEMV_TYPES = (T_QKV, T_OPROJ, T_GATEUP, T_DOWN, T_LMHEAD)
STREAM_TYPES = GEMV_TYPES + (T_DOWNK,)   # tasks that own a run of the packed weight stream
TYPE_NAMES = {T_QKV: "qkv", T_ATTN: "attn", T_MERGE: "merge", T_OPROJ: "oproj", T_GATEUP: "gateup",
              T_DOWN: "down", T_LMHEAD: "lmhead", T_DOWNK: "downk", T_HRED: "hred"}

# field indices inside a task record
F_TYPE, F_LAYER, F_A, F_B, F_K, F_KCHUNKS, F_RT, F_KTC, F_NTILES, F_NKTILES, \
    F_WOFF, F_GEOM, F_R12, F_R13, F_R14, F_AUX = range(16)


class ScheduleError(ValueError):
    """The schedule cannot be executed by the kernel (geometry / smem)."""


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class KernelSchedule:
    """Pipeline parameters of the persistent kernel, taken from the plan."""

    consumer_warps: int = 8
    n_stage: int = 5
    rows_per_tile: int = 64   # plan tile block_n: rows of a tile of the wide operators (gate/up, LM head)
    ktile_chunks: int = 1     # plan tile sub_k / 256; ring slot = rows_per_tile * sub_k * 2 bytes
    attn_min_chunk: int = 128  # positions per split-KV unit before more SMs are used
    inflight: int = 0         # ring stages the Loader keeps in flight at most (0 = all free slots)
    poll_sleep_ns: int = 0    # back-off between polls of an incomplete activation vector
    l2_prefetch_kb: int = 0   # per-SM window past the ring the Loader prefetches into L2 while it is blocked
    poll_inflight: int = 0    # while this SM's consumers poll for inputs: 1-8 = ring stages in flight and no L2 prefetch;
                              # 9 = no new ring fills (their data would return to this SM ahead of the poll replies), L2
                              # prefetch continues; 0 = the Loader ignores the consumers' state
    pace_clk_per_64k: int = 0  # Loader pacing: SM clocks per 64 KB of new HBM requests per SM (0 = unpaced); see pace_for()
    w4a16: bool = False       # the layer projections stream GPTQ-format int4 codes + fp16 group scales (W[n][k] = (q - 8) * s[n][k / 128],
                              # reference byte model graph_ir.py:296-318); needs fuse_down; embedding / LM head stay bf16
    fuse_down: bool = False   # gate/up keeps its SwiGLU outputs on the SM and multiplies them by its own K-slice of the down projection (T_DOWNK);
                              # the 1/n_sms partial rows are summed by T_HRED tasks (no gather of the I-long activation vector)
    stream_down: bool = True  # the down projection streams its input vector in k-tile by k-tile (cp.async) instead of gathering it up front

    def __post_init__(self) -> None:
        if self.consumer_warps not in (4, 7, 8, 16):
            raise ScheduleError("consumer_warps must be 4, 7, 8 or 16")
        if not 2 <= self.n_stage <= MAX_STAGES:
            raise ScheduleError(f"n_stage must be in 2..{MAX_STAGES}")
        if self.rows_per_tile % self.consumer_warps:
            raise ScheduleError("rows_per_tile (block_n) must be a multiple of consumer_warps")
        rw = self.rows_per_tile // self.consumer_warps
        if rw not in (2, 4, 6, 8):
            # an odd count would split a gate/up row pair across warps (SwiGLU is fused in-warp)
            raise ScheduleError("block_n / consumer_warps must be 2, 4, 6 or 8")
        if self.ktile_chunks < 1:
            raise ScheduleError("sub_k must be a positive multiple of 256")
        if self.attn_min_chunk < 8:
            raise ScheduleError("attn_min_chunk out of range")
        if not 0 <= self.inflight <= self.n_stage:
            raise ScheduleError("inflight must be in 0..n_stage")
        if self.w4a16 and not self.fuse_down:
            raise ScheduleError("w4a16 needs fuse_down (the int4 down projection is the fused K-slice kernel)")
        if not 0 <= self.l2_prefetch_kb <= 0xFFFF or not 0 <= self.pace_clk_per_64k <= 0x7FFF:
            raise ScheduleError("l2_prefetch_kb / pace_clk_per_64k out of range")

    @property
    def rows_per_warp(self) -> int:
        return self.rows_per_tile // self.consumer_warps

    @property
    def stage_bytes(self) -> int:
        return self.rows_per_tile * self.ktile_chunks * KCHUNK * 2

    @classmethod
    def from_plan(cls, plan: dict, cfg: "ModelConfig | None" = None, n_sms: int = 148, **overrides) -> "KernelSchedule":
        """Lower ``SolidifiedTrace.plan`` (reference ``search.py:138-171``) to the kernel's pipeline parameters.

        * ``tile`` = [block_m, block_n, block_k, k_split]: a ring stage holds ``rows x sub_k`` weights with
          ``sub_k = block_k / k_split`` and ``rows`` the rows a grid of ``consumer_warps`` warps covers inside the plan
          tile with an even number of rows per warp (gate/up pairs stay in one warp): ``block_n`` rounded down to a
          multiple of ``2 * consumer_warps``, halved while a warp would hold more than eight rows.
        * ``stride_eff``: the planner lets fill ``j`` issue once iteration ``j - stride_eff`` has started (reference
          ``planner.py:583-613``), i.e. ``stride_eff + 1`` stages are in flight at most -> the Loader's ``inflight`` cap.
        * ``n_stage`` / ``per_stage`` / ``window`` / ``pages_required``: the plan is valid on any ring that holds its
          window of ``n_stage`` stages.  The ring's real depth comes from Eq.1 / Eq.2 (reference ``hwmodel.py:207-237``)
          evaluated on the kernel's own shared-memory accounting (``ring_depth``) when ``cfg`` is given; a plan whose
          window does not fit is rejected.
        Run-time knobs the planner does not model (split-KV chunk, L2 prefetch window, fused down projection) come as
        ``overrides``."""
        bm, bn, bk, ks = plan["tile"]
        sub_k = bk // ks
        if sub_k % KCHUNK:
            raise ScheduleError(f"sub_k={sub_k} is not a multiple of {KCHUNK}")
        c = int(plan["consumer_warps"])
        rows = (int(bn) // (2 * c)) * 2 * c
        if rows < 2 * c:
            raise ScheduleError(f"block_n={bn} holds fewer than two rows per consumer warp")
        while rows > MAX_RW * c:     # a plan tile taller than eight rows per warp is executed as several kernel tiles
            rows //= 2
            rows -= rows % (2 * c)
        n_plan = int(plan["n_stage"])
        window, per_stage = int(plan.get("window", 0)), int(plan.get("per_stage", 0))
        if window and per_stage and window != n_plan * per_stage:
            raise ScheduleError("plan window is not n_stage * per_stage pages")
        if "pages_required" in plan and window and int(plan["pages_required"]) < window:
            raise ScheduleError("plan pages_required is smaller than its stream window")
        kw = dict(consumer_warps=c, n_stage=n_plan, rows_per_tile=rows, ktile_chunks=sub_k // KCHUNK,
                  inflight=min(n_plan, int(plan.get("stride_eff", n_plan - 1)) + 1))
        kw.update(overrides)
        sched = cls(**kw)
        if cfg is not None and "n_stage" not in overrides:
            depth = ring_depth(cfg, sched, n_sms=n_sms)
            if depth < n_plan:
                raise ScheduleError(f"the plan's window of {n_plan} stages does not fit the kernel's ring (Eq.2 gives {depth})")
            depth = min(depth, 8)
            sched = cls(**dict(kw, n_stage=depth, inflight=min(kw["inflight"], depth)))
        return sched


RING_PAGE = 1024   # the kernel carves its ring out of shared memory in 1 KB pages (stage_bytes % 1024 == 0)


def ring_depth(cfg: ModelConfig, sched: KernelSchedule, batch: int = 1, n_sms: int = 148) -> int:
    """Ring depth by the paper's constraint model on the kernel's own numbers: Eq.1 gives the pages left after the
    per-CTA overhead (instruction buffer = task cache, semaphores = barrier header, scratch), Eq.2 divides them by
    the pages one stage occupies (reference ``hwmodel.py:207-237``, ``PAPER.md:99-109``)."""
    from .mkplan.hwmodel import HardwareSpec, compute_page_budget, compute_stage_count

    spec = HardwareSpec(smem_max=SMEM_MAX, page_size=RING_PAGE,
                        instr_buf=task_cache_bytes(cfg, batch, n_sms, sched.fuse_down), semaphores=SMEM_RESERVED,
                        scratch=scratch_bytes(cfg, sched, batch, n_sms))
    total = compute_page_budget(spec, 1)                 # the overhead is per CTA, not per stage: N_stage = 1 in Eq.1
    per_stage = _ceil_div(sched.stage_bytes, RING_PAGE)
    return min(MAX_STAGES, compute_stage_count(total, 0, 0, 0, per_stage))


def pace_for(hbm_gbs: float, n_sms: int = 148, sm_mhz: float = 1965.0) -> int:
    """``pace_clk_per_64k`` that meters the Loaders of ``n_sms`` SMs to ``hbm_gbs`` GB/s in aggregate."""
    if hbm_gbs <= 0:
        return 0
    bytes_per_clk = hbm_gbs * 1e9 / n_sms / (sm_mhz * 1e6)
    return max(1, min(0x7FFF, round(65536 / bytes_per_clk)))


def scratch_bytes(cfg: ModelConfig, sched: KernelSchedule, batch: int = 1, n_sms: int = 148) -> int:
    """Shared-memory scratch: the fp32 activation vector of the widest GEMV, or
    the attention unit's q / probability / cross-warp merge buffers."""
    fused = sched.fuse_down and batch == 1
    ks = (cfg.hidden, cfg.q_dim) if fused else (cfg.hidden, cfg.q_dim, cfg.intermediate)   # fused: nobody gathers the I-long vector
    kpad_max = max(_ceil_div(k, KCHUNK) * KCHUNK for k in ks)
    x_bytes = batch * kpad_max * 4
    d = cfg.head_dim
    attn_bytes = ((d + 16) + 2 * d + ATTN_WARPS * (d + 2) + ATTN_WARPS) * 4
    # streamed down projection (csrc: down_streamed): two fp32 slices + four raw tagged-word slices of one k-tile
    stream_bytes = 0
    if sched.stream_down and batch == 1 and not fused:
        _, wk, _, ktc = op_geometry(sched, _ceil_div(cfg.hidden, n_sms), _ceil_div(cfg.intermediate, KCHUNK), False)
        if wk == 1 and ktc * KCHUNK * 40 <= x_bytes + 8192:
            stream_bytes = ktc * KCHUNK * 40
    fused_bytes = fused_scratch_bytes(cfg, n_sms) if fused else 0
    return _ceil_div(max(x_bytes, attn_bytes, stream_bytes, fused_bytes), 1024) * 1024


def fused_scratch_bytes(cfg: ModelConfig, n_sms: int) -> int:
    """Scratch the fused down projection needs: the staged gate/up input (H fp32) followed by this SM's SwiGLU
    outputs (T_DOWNK), or the [rows][n_sms + 1] partial sums a T_HRED task adds up."""
    kpad_h = _ceil_div(cfg.hidden, KCHUNK) * KCHUNK
    act_loc = _ceil_div(cfg.intermediate, n_sms) + 1
    quads = _ceil_div(cfg.hidden // 4, n_sms)
    return max(kpad_h * 4 + act_loc * 4, quads * 4 * hred_stride(n_sms) * 4)


def hred_stride(n_sms: int) -> int:
    """Row stride (floats) of the T_HRED staging array."""
    return n_sms + 1


def task_cache_bytes(cfg: ModelConfig, batch: int = 1, n_sms: int = 148, fused: bool = False) -> int:
    """Shared-memory copy of one SM's task list (32 bytes per task): per layer four GEMV operators (five tasks
    with the fused down projection) plus the attention units and merge tasks placed on the busiest SM; one LM-head task."""
    nq = cfg.n_q_heads
    attn_chunks = max(1, min(n_sms // (batch * nq), ATTN_CHUNKS_MAX))
    per_layer = (5 if fused else 4) + _ceil_div(batch * nq * attn_chunks, n_sms) + _ceil_div(batch * nq, n_sms)
    return _ceil_div((cfg.n_layers * per_layer + 1) * 32, 512) * 512


def max_stages_that_fit(cfg: ModelConfig, sched: KernelSchedule, batch: int = 1, n_sms: int = 148) -> int:
    return ring_depth(cfg, sched, batch, n_sms)


def fuse_down_error(cfg: ModelConfig, sched: KernelSchedule, n_sms: int = 148, tp_size: int = 1) -> str | None:
    """Why the fused down projection (T_DOWNK / T_HRED) cannot run for this model / SM count, or None."""
    if tp_size != 1:
        return "fuse_down is a single-GPU schedule (tensor-parallel ranks publish partial rows to their peers instead)"
    if cfg.hidden % 256:
        return "fuse_down needs hidden to be a multiple of 256 (eight rows per lane, 32 lanes)"
    if _ceil_div(cfg.hidden // 256, sched.consumer_warps) > 3:
        return "fuse_down: more than three 256-row blocks per consumer warp"
    if sched.stage_bytes < cfg.hidden * 2:
        return "fuse_down: a ring slot must hold one column of the down projection"
    if _ceil_div(cfg.hidden // 4, n_sms) > 16:
        return "fuse_down: more than 16 row quads per T_HRED task"
    if cfg.intermediate < n_sms:
        return "fuse_down: every SM must own at least one gate/up pair (its partial rows are awaited by every T_HRED task)"
    return None


def split_rows(n_units: int, n_sms: int, rot: int) -> list[tuple[int, int]]:
    """Contiguous, near-even split of ``n_units`` over ``n_sms`` SMs.

    The ``n_units % n_sms`` SMs that take one extra unit start at SM ``rot`` so
    consecutive operators put their remainder on different SMs and the per-SM
    byte streams stay balanced.  Returns [(first_unit, count)] indexed by SM."""
    base, rem = divmod(n_units, n_sms)
    out = [(0, 0)] * n_sms
    for jr in range(n_sms):
        sm = (jr + rot) % n_sms
        first = jr * base + min(jr, rem)
        out[sm] = (first, base + (1 if jr < rem else 0))
    return out


def op_geometry(sched: KernelSchedule, max_rows: int, kchunks: int, pairs: bool, chunk_row_bytes: int = KCHUNK * 2) -> tuple[int, int, int, int]:
    """Warp grid of one operator: (WR, WK, rows per warp, chunks per stage).

    The C consumer warps form WR row groups x WK interleaved K groups.  Wide
    operators (more rows per SM than a K-split tile holds) use the plan tile:
    WR = C, WK = 1, ``rows_per_tile`` rows.  Narrow operators (10-14 rows per SM
    for the 1.5B projections) would leave most warps idle that way, so they
    split K across warps instead; the split with the least per-warp work
    (row-chunk iterations + per-stage overhead) wins, ties to fewer stages."""
    c = sched.consumer_warps

    def plan_tile():
        # rows per warp: at most the plan tile's, chosen so the last tile of the SM's slice is not mostly
        # padding (122 gate/up rows on 7 warps: three 56-row tiles are 73 % full, three 42-row tiles 97 %)
        best_rw, best_pad = sched.rows_per_warp, None
        for rw in range(sched.rows_per_warp, 0, -1):
            if rw & 1:
                continue
            rt = c * rw
            n_t = _ceil_div(max_rows, rt)
            # row slots computed (padding included) + ~8 rows' worth of reduce / epilogue per tile, scaled by
            # the activation-load overhead of short row groups (2 LDS.128 of x per rw of weights)
            cost = (n_t * rt + 8 * n_t) * (1.0 + 1.0 / rw)
            if best_pad is None or cost < best_pad:
                best_rw, best_pad = rw, cost
        rw = best_rw
        rt = c * rw
        ktc = max(1, min(kchunks, sched.stage_bytes // (rt * chunk_row_bytes)))
        n_kt = _ceil_div(kchunks, ktc)
        return c, 1, rw, _ceil_div(kchunks, n_kt)

    if max_rows > c * MAX_RW:
        return plan_tile()
    best = None
    wk = 1
    while wk <= c:
        if c % wk:
            wk *= 2
            continue
        wr = c // wk
        rw = _ceil_div(max_rows, wr)
        rw += rw & 1     # the kernel's row loops are instantiated for 2, 4, 6, 8 rows per warp: keep rt = WR * rw honest
                         # about the rows a warp touches (and gate/up pairs inside one warp)
        rt = wr * rw
        if rw <= MAX_RW and (wk == 1 or rt <= 32):
            ktc_max = min(kchunks, sched.stage_bytes // (rt * chunk_row_bytes))
            for ktc in range(1, ktc_max + 1):
                n_kt = _ceil_div(kchunks, ktc)
                ktc_e = _ceil_div(kchunks, n_kt)
                cost = 3 if wk > 1 else 0
                for kt in range(n_kt):
                    ch = min(ktc_e, kchunks - kt * ktc_e)
                    cost += _ceil_div(ch, wk) * (rw + 1) + 2
                key = (cost, n_kt, wk)
                if best is None or key < best[0]:
                    best = (key, (wr, wk, rw, ktc_e))
        wk *= 2
    if best is None:   # the ring slot is too small for a single tile of all rows: several plan tiles
        return plan_tile()
    return best[1]


@dataclass
class TaskTable:
    cfg: ModelConfig
    sched: KernelSchedule
    n_sms: int
    batch: int
    header: np.ndarray      # int32[HEADER_INTS]
    sm_begin: np.ndarray    # int32[n_sms + 1]
    tasks: np.ndarray       # int32[n_tasks, TASK_INTS]
    packed_weight_bytes: int
    attn_chunks: int

    @property
    def blob(self) -> bytes:
        return np.concatenate([self.header, self.sm_begin, self.tasks.reshape(-1)]).astype("<i4").tobytes()

    def tasks_of(self, sm: int) -> np.ndarray:
        return self.tasks[self.sm_begin[sm]:self.sm_begin[sm + 1]]

    def stream_bytes_per_sm(self) -> np.ndarray:
        out = np.zeros(self.n_sms, dtype=np.int64)
        for sm in range(self.n_sms):
            out[sm] = sum(task_weight_bytes(t) for t in self.tasks_of(sm))
        return out

    def summary(self) -> dict:
        per_sm = self.stream_bytes_per_sm()
        return {
            "n_sms": self.n_sms, "n_tasks": int(self.tasks.shape[0]),
            "consumer_warps": self.sched.consumer_warps, "n_stage": self.sched.n_stage,
            "stage_bytes": self.sched.stage_bytes, "packed_weight_bytes": int(self.packed_weight_bytes),
            "stream_bytes_min": int(per_sm.min()), "stream_bytes_max": int(per_sm.max()),
            "attn_chunks": self.attn_chunks,
        }


def stage_shapes(task: np.ndarray):
    """Yield (tile, ktile, rows, chunks) for every ring stage of a GEMV task, in
    the order the Loader issues them and the Consumers drain them."""
    nrows, rt, ktc, kchunks = int(task[F_B]), int(task[F_RT]), int(task[F_KTC]), int(task[F_KCHUNKS])
    for tile in range(int(task[F_NTILES])):
        rows = min(rt, nrows - tile * rt)
        for kt in range(int(task[F_NKTILES])):
            yield tile, kt, rows, min(ktc, kchunks - kt * ktc)


I4_GROUP = 128           # reduction elements per fp16 scale (reference graph_ir.INT4_GROUP_SIZE)
I4_CHUNK_BYTES = 128     # a 256-element chunk of one row as 4-bit codes
I4_SCALE_BYTES = 4       # its two fp16 scales
AUX_LOCAL_ACT, AUX_INT4 = 1, 2


def i4_stage_bytes(rows: int, chunks: int) -> int:
    return (rows * chunks * (I4_CHUNK_BYTES + I4_SCALE_BYTES) + 15) & ~15


def downk_i4_groups(k0: int, nk: int) -> int:
    return (k0 + nk - 1) // I4_GROUP - k0 // I4_GROUP + 1


def task_weight_bytes(task) -> int:
    """Bytes of the packed weight stream a task owns (csrc/adamk.cu: task_stream_bytes)."""
    ttype, i4 = int(task[F_TYPE]), bool(int(task[F_AUX]) & AUX_INT4)
    if ttype == T_DOWNK:      # b columns of the down projection, k = H rows each (+ the fp16 scales of the groups they touch)
        b, h = int(task[F_B]), int(task[F_K])
        return downk_i4_groups(int(task[F_A]), b) * h * 2 + b * h // 2 if i4 else b * h * 2
    if ttype not in GEMV_TYPES:
        return 0
    if not i4:                # rows * kchunks * 512, independent of tiling
        return int(task[F_B]) * int(task[F_KCHUNKS]) * KCHUNK * 2
    return sum(i4_stage_bytes(rows, chunks) for _, _, rows, chunks in stage_shapes(task))


def unpack_geom(geom: int) -> tuple[int, int, int]:
    return geom & 0xFF, (geom >> 8) & 0xFF, (geom >> 16) & 0xFF


def build_task_table(cfg: ModelConfig, sched: KernelSchedule, n_sms: int = 148, batch: int = 1) -> TaskTable:
    if batch != 1:
        raise ScheduleError("this build executes batch 1 only (batched path: SURVEY.md 8(f).1)")
    if n_sms < 1:
        raise ScheduleError("n_sms must be >= 1")
    fit = max_stages_that_fit(cfg, sched, batch, n_sms)
    if sched.n_stage > fit:
        raise ScheduleError(
            f"n_stage={sched.n_stage} x {sched.stage_bytes} B stages + "
            f"{scratch_bytes(cfg, sched, batch, n_sms)} B scratch exceed {SMEM_MAX} B shared memory (max {fit})")
    if sched.stage_bytes < 8 * min(sched.consumer_warps, ATTN_WARPS) * cfg.head_dim * 2:
        raise ScheduleError("ring slot smaller than one 64-position K/V block")
    if cfg.group > G_MAX:
        raise ScheduleError(f"more than {G_MAX} q heads per kv head")
    for k in (cfg.hidden, cfg.q_dim, cfg.intermediate):
        if k % 8:
            raise ScheduleError("reduction dims must be multiples of 8")

    nq = cfg.n_q_heads
    attn_chunks = max(1, min(n_sms // (batch * nq), ATTN_CHUNKS_MAX))
    per_sm: list[list[list[int]]] = [[] for _ in range(n_sms)]
    rot = 0

    fuse, i4 = sched.fuse_down, sched.w4a16
    if i4 and any(k % 8 for k in (cfg.hidden, cfg.q_dim, cfg.intermediate)):
        raise ScheduleError("w4a16: reduction dims must be multiples of 8")
    if fuse:
        why = fuse_down_error(cfg, sched, n_sms)
        if why:
            raise ScheduleError(why)

    def gemv(ttype: int, layer: int, n_rows: int, k: int, unit: int, aux: int = 0) -> int:
        """Emit one GEMV operator across all SMs; returns the number of tasks."""
        nonlocal rot
        assert n_rows % unit == 0
        kchunks = _ceil_div(k, KCHUNK)
        split = split_rows(n_rows // unit, n_sms, rot)
        rot = (rot + (n_rows // unit) % n_sms) % n_sms
        max_rows = max(cnt for _, cnt in split) * unit
        int4_op = i4 and ttype != T_LMHEAD
        wr, wk, rw, ktc = op_geometry(sched, max_rows, kchunks, pairs=(unit == 2),
                                      chunk_row_bytes=(I4_CHUNK_BYTES + I4_SCALE_BYTES + 1) if int4_op else KCHUNK * 2)
        rt = wr * rw
        n_kt = _ceil_div(kchunks, ktc)
        geom = wr | (wk << 8) | (rw << 16)
        emitted = 0
        for sm, (first, cnt) in enumerate(split):
            if cnt == 0:
                continue
            nrows = cnt * unit
            n_tiles = _ceil_div(nrows, rt)
            per_sm[sm].append([ttype, layer, first * unit, nrows, k, kchunks, rt, ktc,
                               n_tiles, n_kt, 0, geom, 0, 0, 0, aux | (AUX_INT4 if i4 and ttype != T_LMHEAD else 0)])
            emitted += 1
            if ttype == T_GATEUP and aux:
                # this SM's K-slice of the down projection: columns first .. first + cnt, all H rows each, column-major;
                # a ring stage holds `cps` whole columns
                cps = max(1, sched.stage_bytes // (cfg.hidden * 2))
                if i4:
                    cps = max(1, sched.stage_bytes // (cfg.hidden // 2))
                    if downk_i4_groups(first, cnt) > 3 or downk_i4_groups(first, cnt) * cfg.hidden * 2 > sched.stage_bytes:
                        raise ScheduleError("w4a16: an SM's slice of the down projection touches too many scale groups")
                per_sm[sm].append([T_DOWNK, layer, first, cnt, cfg.hidden, cps, 0, 0, 1, _ceil_div(cnt, cps),
                                   0, 0, 0, 0, 0, AUX_INT4 if i4 else 0])
        return emitted

    def hred(layer: int) -> None:
        """Sum the n_sms partial rows of the fused down projection (+ residual): row quads split over the SMs."""
        nonlocal rot
        nquads = cfg.hidden // 4
        split = split_rows(nquads, n_sms, rot)
        rot = (rot + nquads % n_sms) % n_sms
        for sm, (first, cnt) in enumerate(split):
            if cnt:
                per_sm[sm].append([T_HRED, layer, first, cnt, cfg.hidden, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0])

    for layer in range(cfg.n_layers):
        gemv(T_QKV, layer, cfg.qkv_rows, cfg.hidden, 1)
        for b in range(batch):
            # one unit per (q head, context chunk): chunk-major so the units that are active at short
            # contexts (chunk 0, 1, ...) land on different SMs
            for c in range(attn_chunks):
                for h in range(nq):
                    sm = ((b * attn_chunks + c) * nq + h) % n_sms
                    per_sm[sm].append([T_ATTN, layer, h, c, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, b])
            # flash-decoding merge of the units of one q head; placed on the SMs whose attention
            # units are the last to become active as the context grows
            for h in range(cfg.n_q_heads):
                sm = (n_sms - 1 - (b * cfg.n_q_heads + h)) % n_sms
                per_sm[sm].append([T_MERGE, layer, h, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, b])
        gemv(T_OPROJ, layer, cfg.hidden, cfg.q_dim, 1)
        if fuse:
            gemv(T_GATEUP, layer, 2 * cfg.intermediate, cfg.hidden, 2, aux=1)
            hred(layer)
        else:
            gemv(T_GATEUP, layer, 2 * cfg.intermediate, cfg.hidden, 2)
            gemv(T_DOWN, layer, cfg.hidden, cfg.intermediate, 1)
    n_lm = gemv(T_LMHEAD, cfg.n_layers, cfg.vocab, cfg.hidden, 1)

    # weight offsets: each SM's stream is one contiguous run, SM-major
    cursor = 0
    sm_begin = np.zeros(n_sms + 1, dtype=np.int32)
    flat: list[list[int]] = []
    for sm in range(n_sms):
        sm_begin[sm] = len(flat)
        for t in per_sm[sm]:
            if t[F_TYPE] in STREAM_TYPES:
                t[F_WOFF] = cursor // 16
                cursor += task_weight_bytes(t)
            flat.append(t)
    sm_begin[n_sms] = len(flat)
    if cursor // 16 >= 2 ** 31:
        raise ScheduleError("packed weights exceed the 32 GiB offset range of the task record")
    tasks = np.asarray(flat, dtype=np.int32).reshape(-1, TASK_INTS)

    header = np.zeros(HEADER_INTS, dtype=np.int32)
    header[:13] = [MAGIC, VERSION, n_sms, sched.consumer_warps, sched.n_stage, sched.stage_bytes,
                   tasks.shape[0], batch, sched.inflight, attn_chunks, sched.attn_min_chunk,
                   scratch_bytes(cfg, sched, batch, n_sms), n_lm]
    header[13] = (cursor // 16) & 0x7FFFFFFF
    header[14] = ((sched.poll_sleep_ns & 0xFFFF) | ((0 if sched.stream_down else 1) << 16) | ((sched.poll_inflight & 0xF) << 20)
                  | ((1 if fuse else 0) << 24) | ((1 if i4 else 0) << 26))
    header[15] = (sched.l2_prefetch_kb & 0xFFFF) | ((sched.pace_clk_per_64k & 0x7FFF) << 16)
    return TaskTable(cfg=cfg, sched=sched, n_sms=n_sms, batch=batch, header=header, sm_begin=sm_begin,
                     tasks=tasks, packed_weight_bytes=cursor, attn_chunks=attn_chunks)


# ---------------------------------------------------------------------------
# Host restatement of the device weight packer (tests: exact-cover + bit parity)
# ---------------------------------------------------------------------------

def virtual_row_source(cfg: ModelConfig, ttype: int, vrow: int) -> tuple[str, int]:
    """(matrix name, row) a virtual output row of an operator reads."""
    if ttype == T_QKV:
        if vrow < cfg.q_dim:
            return "wq", vrow
        if vrow < cfg.q_dim + cfg.kv_dim:
            return "wk", vrow - cfg.q_dim
        return "wv", vrow - cfg.q_dim - cfg.kv_dim
    if ttype == T_OPROJ:
        return "wo", vrow
    if ttype == T_GATEUP:      # gate/up rows interleaved so one warp owns a pair
        return ("wup", vrow >> 1) if vrow & 1 else ("wgate", vrow >> 1)
    if ttype == T_DOWN:
        return "wdown", vrow
    if ttype == T_LMHEAD:
        return "lm_head", vrow
    raise ValueError(ttype)


def chunk_permutation() -> np.ndarray:
    """Packed position -> original offset inside one 256-element K chunk.

    Lane ``l`` owns packed elements ``8l..8l+7``; they hold original offsets
    ``4l..4l+3`` and ``128+4l..128+4l+3`` so that the matching fp32 activations
    are two conflict-free LDS.128 per lane."""
    p = np.arange(KCHUNK)
    lane, e = p // 8, p % 8
    return (e >> 2) * 128 + lane * 4 + (e & 3)


def pack_weights_reference(table: TaskTable, weights) -> np.ndarray:
    """NumPy restatement of ``adamk_pack_kernel``: uint16 view of the packed bf16
    weight stream (without the fp32 parameter tail)."""
    import torch

    cfg = table.cfg
    perm = chunk_permutation()
    out = np.zeros(table.packed_weight_bytes // 2, dtype=np.uint16)

    def as_u16(t):
        return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)

    mats: dict[tuple[int, str], np.ndarray] = {}

    def mat(layer: int, name: str) -> np.ndarray:
        key = (layer, name)
        if key not in mats:
            if name == "lm_head":
                mats[key] = as_u16(weights.lm_head_matrix)
            else:
                mats[key] = as_u16(getattr(weights.layers[layer], name))
        return mats[key]

    qlayers = getattr(weights, "layers", None) if hasattr(weights, "base") else None     # quant.QuantizedWeights
    if qlayers is not None:
        weights_q, weights = weights, weights.base
        out8 = out.view(np.uint8)

        def code(qm, row: int, kidx: np.ndarray, k: int) -> np.ndarray:
            b = qm.q[row].cpu().numpy()[np.minimum(kidx, k - 1) // 2]
            return np.where(kidx < k, np.where(kidx & 1, b >> 4, b & 15), 8).astype(np.uint8)

    for task in table.tasks:
        ttype = int(task[F_TYPE])
        if qlayers is not None and int(task[F_AUX]) & AUX_INT4:
            layer, pos = int(task[F_LAYER]), int(task[F_WOFF]) * 16   # bytes
            ql = qlayers[layer]
            if ttype == T_DOWNK:
                k0, nk, h = int(task[F_A]), int(task[F_B]), int(task[F_K])
                qm = ql["wdown"]
                g0, ng = k0 // I4_GROUP, downk_i4_groups(k0, nk)
                sc = qm.s.cpu().numpy().view(np.uint16)[:, g0:g0 + ng].T.reshape(-1)          # [group][row]
                out8[pos:pos + ng * h * 2] = sc.astype("<u2").view(np.uint8)
                pos += ng * h * 2
                qb = qm.q.cpu().numpy()
                for j in range(nk):
                    kk = k0 + j
                    col = (qb[:, kk // 2] >> 4) if kk & 1 else (qb[:, kk // 2] & 15)            # codes of all rows
                    out8[pos:pos + h // 2] = (col[0::2] | (col[1::2] << 4)).astype(np.uint8)
                    pos += h // 2
                continue
            vrow0, k, rt, ktc = int(task[F_A]), int(task[F_K]), int(task[F_RT]), int(task[F_KTC])
            lane = np.arange(32)
            for tile, kt, rows, chunks in stage_shapes(task):
                stage = np.zeros(i4_stage_bytes(rows, chunks), dtype=np.uint8)
                scales = np.zeros(rows * chunks * 2, dtype=np.uint16)
                for r in range(rows):
                    name, row = virtual_row_source(cfg, ttype, vrow0 + tile * rt + r)
                    qm = ql[name]
                    srow = qm.s[row].cpu().numpy().view(np.uint16)
                    for c in range(chunks):
                        kbase = (kt * ktc + c) * KCHUNK
                        blk = r * chunks + c
                        words = np.zeros(32, dtype=np.uint32)
                        for el in range(8):
                            kidx = kbase + (4 * lane + el if el < 4 else 128 + 4 * lane + el - 4)
                            words |= code(qm, row, kidx, k).astype(np.uint32) << (4 * el)
                        stage[blk * I4_CHUNK_BYTES:(blk + 1) * I4_CHUNK_BYTES] = words.astype("<u4").view(np.uint8)
                        for gi in range(2):
                            g = kbase // I4_GROUP + gi
                            scales[blk * 2 + gi] = srow[g] if g < srow.size else 0
                stage[rows * chunks * I4_CHUNK_BYTES:rows * chunks * (I4_CHUNK_BYTES + I4_SCALE_BYTES)] = scales.astype("<u2").view(np.uint8)
                out8[pos:pos + stage.size] = stage
                pos += stage.size
            continue
        if ttype == T_DOWNK:   # columns k0 .. k0 + nk of the down projection, each as H consecutive rows
            k0, nk = int(task[F_A]), int(task[F_B])
            pos = int(task[F_WOFF]) * 8
            src = mat(int(task[F_LAYER]), "wdown")           # [H, I]
            blk = np.ascontiguousarray(src[:, k0:k0 + nk].T).reshape(-1)
            out[pos:pos + blk.size] = blk
            continue
        if ttype not in GEMV_TYPES:
            continue
        layer, vrow0, k = int(task[F_LAYER]), int(task[F_A]), int(task[F_K])
        rt, ktc = int(task[F_RT]), int(task[F_KTC])
        pos = int(task[F_WOFF]) * 8  # uint16 elements
        for tile, kt, rows, chunks in stage_shapes(task):
            for r in range(rows):
                name, row = virtual_row_source(cfg, ttype, vrow0 + tile * rt + r)
                src = mat(layer, name)[row]
                for c in range(chunks):
                    kbase = (kt * ktc + c) * KCHUNK
                    kidx = kbase + perm
                    vals = np.where(kidx < k, src[np.minimum(kidx, k - 1)], 0).astype(np.uint16)
                    out[pos:pos + KCHUNK] = vals
                    pos += KCHUNK
    return out
