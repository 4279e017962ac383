"""Solidified kernel schedules shipped with the package.

``default_schedule`` returns the ring parameters the plugin uses when the caller
does not supply a SolidifiedTrace of their own.  The values are read from the
plan files under ``schedules/`` -- ``mkplan search`` output for the per-layer
operator graph on ``fixtures/b200.json`` -- when one exists for the model, and
otherwise fall back to the profiled default below (offline profiling on the
target GPU is how the paper locks in its trace).
"""

from __future__ import annotations

from pathlib import Path

from .model_config import ModelConfig
from dataclasses import replace

from .task_table import KernelSchedule, fuse_down_error, max_stages_that_fit

SCHEDULE_DIR = Path(__file__).resolve().parent / "schedules"

# Profiled on B200 (profiles/): 7 consumer warps + the Loader warp = 8 warps per CTA (the register
# file then gives every thread 255 registers; 9 warps are capped at 168 and the GEMV loop spills),
# 42-row x 512-column sub-tiles (42 KB ring slots, four of them: two chunk iterations per warp per stage
# amortise the per-stage barrier work, and 42 rows tile the 120-122 gate/up rows of an SM without padding), ring as deep as shared memory allows, 112-position split-KV units (two 56-position K/V blocks: one pass of the seven warps each),
# and a 512 KB per-SM L2 prefetch window past the ring.
PROFILED_DEFAULT = dict(consumer_warps=7, rows_per_tile=42, ktile_chunks=2, attn_min_chunk=112, l2_prefetch_kb=512, fuse_down=True)


def default_schedule(cfg: ModelConfig, n_sms: int = 148, tp_size: int = 1) -> KernelSchedule:
    """The model's shipped SolidifiedTrace (``schedules/<model>.trace.json``, written by ``mkplan search`` through
    ``tools/make_schedules.py``) lowered to the kernel; models without one fall back to the profiled default."""
    from .solidify import schedule_from_trace, shipped_trace

    shipped = shipped_trace(cfg)
    if shipped is not None:
        trace, knobs, _ = shipped
        return schedule_from_trace(cfg, trace, knobs, n_sms, tp_size)
    return fit_schedule(cfg, KernelSchedule(n_stage=2, **PROFILED_DEFAULT), n_sms, tp_size)


def schedule_id(cfg: ModelConfig) -> dict:
    """What the bench line reports about the schedule in use."""
    from .solidify import shipped_trace

    shipped = shipped_trace(cfg)
    if shipped is None:
        return {"source": "profiled default (no solidified trace shipped for this model)"}
    trace, knobs, order = shipped
    return {"source": f"mkplan search -> schedules/{cfg.name}.trace.json", "content_hash": trace.content_hash,
            "tile": trace.plan["tile"], "plan_n_stage": trace.plan["n_stage"], "stride_eff": trace.plan["stride_eff"],
            "kernel_knobs": knobs, "program_order_checked": order is not None}


def fit_schedule(cfg: ModelConfig, sched: KernelSchedule, n_sms: int = 148, tp_size: int = 1, keep_fused: bool = False) -> KernelSchedule:
    """Adapt a schedule to a model / SM count: the fused down projection only where it can run -- and, unless
    ``keep_fused`` (or the schedule is W4A16, which needs it), only where it pays --, the ring as deep as shared memory
    allows (at most eight stages), at most three stages in flight (a fourth only lengthens the queue every tagged-word
    poll waits behind)."""
    if sched.fuse_down:
        impossible = fuse_down_error(cfg, sched, n_sms, tp_size)
        # where it pays: one 256-row block per consumer warp (measured, tools/model_sweep.py: Qwen2.5-1.5B 811 vs 822
        # us/token fused vs not; with two or three blocks per warp the K-slice kernel loses its balance: Qwen2.5-7B
        # 2511 vs 2498, Qwen3-8B 2724 vs 2628)
        unprofitable = cfg.hidden // 256 > sched.consumer_warps and not (keep_fused or sched.w4a16)
        if impossible or unprofitable:
            sched = replace(sched, fuse_down=False, w4a16=False)
    n_stage = max(2, min(max_stages_that_fit(cfg, replace(sched, n_stage=2, inflight=0), n_sms=n_sms), 8))
    return replace(sched, n_stage=n_stage, inflight=min(3, n_stage))
