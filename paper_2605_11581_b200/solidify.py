"""SolidifiedTrace -> kernel schedule: the glue between the offline search and the persistent kernel.

The reference's artifact (``pkg/src/mkplan/search.py:79-171``) carries, for ONE SM running ONE layer's pipeline,
the tile, pipeline depth, consumer-warp count, prefetch stride, the per-role programs ``[[op_id, start, finish], ...]``
and the page plan.  The kernel replays a fixed order per SM -- operators in graph order; inside a weight-streaming
operator the Loader fills (row tile, k tile) stages tile-major and the Consumers drain them in that order
(csrc/adamk.cu: the Loader loop / gemv_ktiles; task_table.stage_shapes).  ``check_program_order`` proves that this IS
the order of the plan's Loader and Consumer programs, so the static task table is the plan's schedule and not merely
parameterised by it; a plan whose passes (gap fill) hoisted work across stages is rejected.

A shipped trace lives in ``schedules/<model>.trace.json`` next to the exact ``.graph.json`` / ``.space.json`` /
``.hw.json`` inputs that reproduce it (``tools/make_schedules.py``; the reference planner gives the same bytes:
``tests/test_schedules.py``) and a ``.kernel.json`` with the run-time knobs the planner does not model.
"""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

from .mkplan.hwmodel import MicroOpKind
from .mkplan.search import SolidifiedTrace, parse_trace, rebuild_candidate
from .model_config import ModelConfig
from .task_table import KernelSchedule, ScheduleError

SCHEDULE_DIR = Path(__file__).resolve().parent / "schedules"


def check_program_order(trace: SolidifiedTrace, graph_text: str, hw_text: str) -> dict:
    """Assert that the plan's Loader / Consumer programs are in the order the kernel replays; returns counts.

    Loader: every fill in micro-op id order = (operator, row tile, k step) order (reference lowering
    ``graph_ir.py:381-452``: ``jn`` outer, ``step`` inner -- the kernel's (tile, kt) stage order).
    Consumer: the stage keys (operator, row tile, k step) along the program never go backwards: the consumers drain
    stage s completely before stage s + 1."""
    from .mkplan.graph_ir import GEMM_LIKE, load_graph

    cand, _ = rebuild_candidate(trace, graph_text, hw_text)
    streaming = {o.id for o in load_graph(graph_text).operators if o.kind in GEMM_LIKE}
    ops = {op.id: op for op in cand.trace.ops}
    op_index: dict[str, int] = {}
    for op in cand.trace.ops:
        op_index.setdefault(op.source_operator, len(op_index))
    programs = trace.plan["programs"]
    loader = [row[0] for row in programs.get("Loader", [])]
    if loader != sorted(loader):
        raise ScheduleError("the plan's Loader program is not in stage order: the kernel's Loader cannot replay it")
    fills = [i for i in loader if ops[i].kind == MicroOpKind.GlobalToShared]
    last = (-1, -1, -1)
    n_stage_keys = 0
    for i in (row[0] for row in programs.get("Consumer", [])):
        op = ops[i]
        coord = tuple(op.tile_coord) + (0,) * (3 - len(op.tile_coord))
        # element-wise operators (norms, SwiGLU, residual adds) are fused into the neighbouring GEMV's prologue /
        # epilogue by the kernel: only their operator order is checked
        key = (op_index[op.source_operator], coord[1], coord[2]) if op.source_operator in streaming else (op_index[op.source_operator], 0, 0)
        if key < last:
            raise ScheduleError(f"the plan's Consumer program hoists micro-op {i} ({op.source_operator} {coord}) ahead of stage "
                                f"{last}: the kernel drains its ring in order and cannot replay it")
        if key != last:
            n_stage_keys += 1
        last = key
    return {"loader_ops": len(loader), "fills": len(fills), "consumer_ops": len(programs.get("Consumer", [])),
            "consumer_stages": n_stage_keys}


@lru_cache(maxsize=None)
def _shipped(name: str):
    f = SCHEDULE_DIR / f"{name}.trace.json"
    if not f.exists():
        return None
    trace = parse_trace(f.read_bytes())     # verifies format version and content hash
    side = SCHEDULE_DIR / f"{name}.kernel.json"
    knobs = json.loads(side.read_text()) if side.exists() else {}
    graph, hw = SCHEDULE_DIR / f"{name}.graph.json", SCHEDULE_DIR / f"{name}.hw.json"
    order = check_program_order(trace, graph.read_text(), hw.read_text()) if graph.exists() and hw.exists() else None
    return trace, knobs, order


def shipped_trace(cfg: ModelConfig):
    """(SolidifiedTrace, kernel knobs, program-order check) of the model's shipped schedule, or None."""
    return _shipped(cfg.name)


def schedule_from_trace(cfg: ModelConfig, trace: SolidifiedTrace, knobs: dict | None = None, n_sms: int = 148,
                        tp_size: int = 1) -> KernelSchedule:
    """The kernel schedule a trace solidifies for this model / SM count (``KernelSchedule.from_plan``), with the
    fused down projection only where it can run."""
    from .task_table import fuse_down_error

    knobs = dict(knobs or {})
    probe = KernelSchedule.from_plan(trace.plan, **knobs)
    if knobs.get("fuse_down") and fuse_down_error(cfg, probe, n_sms, tp_size):
        knobs["fuse_down"] = False
    return KernelSchedule.from_plan(trace.plan, cfg, n_sms, **knobs)
