"""Solidified kernel schedules shipped with the package.

``default_schedule`` returns the ring parameters the plugin uses when the caller
does not supply a SolidifiedTrace of their own.  The values are read from the
plan files under ``schedules/`` -- ``mkplan search`` output for the per-layer
operator graph on ``fixtures/b200.json`` -- when one exists for the model, and
otherwise fall back to the profiled default below (offline profiling on the
target GPU is how the paper locks in its trace).
"""

from __future__ import annotations

import json
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
    plan_file = SCHEDULE_DIR / f"{cfg.name}.trace.json"
    if plan_file.exists():
        plan = json.loads(plan_file.read_text())["plan"]
        sched = KernelSchedule.from_plan(plan)
        fit = max_stages_that_fit(cfg, sched, n_sms=n_sms)
        if sched.n_stage > fit:
            sched = KernelSchedule.from_plan(plan, n_stage=fit)
        return sched
    return fit_schedule(cfg, KernelSchedule(n_stage=2, **PROFILED_DEFAULT), n_sms, tp_size)


def fit_schedule(cfg: ModelConfig, sched: KernelSchedule, n_sms: int = 148, tp_size: int = 1) -> KernelSchedule:
    """Adapt a schedule to a model / SM count: the fused down projection only where it can run, the ring as deep as
    shared memory allows (at most eight stages), at most three stages in flight (a fourth only lengthens the queue
    every tagged-word poll waits behind)."""
    if sched.fuse_down and fuse_down_error(cfg, sched, n_sms, tp_size):
        sched = replace(sched, fuse_down=False)
    n_stage = max(2, min(max_stages_that_fit(cfg, replace(sched, n_stage=2, inflight=0), n_sms=n_sms), 8))
    return replace(sched, n_stage=n_stage, inflight=min(3, n_stage))
