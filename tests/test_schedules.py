"""The shipped SolidifiedTrace drives the kernel (CPU only).

* the trace file is a genuine ``mkplan search`` output: this repository's planner AND the reference planner
  (``/root/reference/pkg/src/mkplan``, when present) reproduce its bytes from the committed graph / hw / space files;
* ``KernelSchedule.from_plan`` consumes tile, consumer_warps, stride_eff, n_stage / per_stage / window /
  pages_required, and derives the ring depth through Eq.1 / Eq.2 on the kernel's shared-memory accounting;
* the plan's Loader / Consumer programs are in the order the kernel replays (``solidify.check_program_order``).
"""

import copy
import json
import sys
from pathlib import Path

import pytest

from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.mkplan import search
from paper_2605_11581_b200.mkplan.hwmodel import HardwareSpec, compute_page_budget, compute_stage_count
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.schedules import default_schedule, schedule_id
from paper_2605_11581_b200.solidify import SCHEDULE_DIR, check_program_order, schedule_from_trace, shipped_trace

REF = Path("/root/reference/pkg/src")
NAME = "qwen2.5-1.5b"
CFG = PRESETS[NAME]


SHIPPED = ("qwen2.5-1.5b", "qwen2.5-7b", "qwen3-8b")


def _files(name=NAME):
    return {k: (SCHEDULE_DIR / f"{name}.{k}.json") for k in ("trace", "graph", "hw", "space", "kernel")}


def test_shipped_trace_is_well_formed_and_hash_checked():
    f = _files()
    for p in f.values():
        assert p.exists(), p
    trace = search.parse_trace(f["trace"].read_bytes())          # raises on a wrong content hash
    assert search.serialize_trace(trace) == f["trace"].read_bytes()
    assert trace.plan["consumer_warps"] == 7 and trace.plan["tile"][0] == 16
    raw = f["trace"].read_bytes()
    bad = raw.replace(b'"n_stage":%d' % trace.plan["n_stage"], b'"n_stage":%d' % (trace.plan["n_stage"] + 1), 1)
    assert bad != raw
    with pytest.raises(search.TraceFormatError):
        search.parse_trace(bad)


@pytest.mark.parametrize("name", SHIPPED)
def test_mirror_planner_reproduces_the_shipped_trace_bytes(name):
    f = _files(name)
    trace = search.run_search(f["graph"].read_text(), f["hw"].read_text(), f["space"].read_text(), 10000)
    assert search.serialize_trace(trace) == f["trace"].read_bytes()


@pytest.mark.skipif(not REF.exists(), reason="the reference planner is only mounted in the build container")
@pytest.mark.parametrize("name", SHIPPED)
def test_reference_planner_reproduces_the_shipped_trace_bytes(name):
    import importlib

    f = _files(name)
    saved = {k: v for k, v in sys.modules.items() if k == "mkplan" or k.startswith("mkplan.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, str(REF))
    try:
        ref_search = importlib.import_module("mkplan.search")
        assert str(REF) in ref_search.__file__
        trace = ref_search.run_search(f["graph"].read_text(), f["hw"].read_text(), f["space"].read_text(), 10000)
        text = ref_search.serialize_trace(trace)
        text = text if isinstance(text, bytes) else text.encode()
        assert text == f["trace"].read_bytes()
    finally:
        sys.path.remove(str(REF))
        for k in [k for k in sys.modules if k == "mkplan" or k.startswith("mkplan.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def test_from_plan_consumes_the_plan_and_derives_the_ring_by_eq1_eq2():
    trace, knobs, order = shipped_trace(CFG)
    plan = trace.plan
    sched = schedule_from_trace(CFG, trace, knobs)
    assert sched == default_schedule(CFG)
    c = plan["consumer_warps"]
    assert sched.consumer_warps == c
    # rows: block_n rounded down to an even number of rows per warp; stage columns: block_k / k_split
    assert sched.rows_per_tile == plan["tile"][1] // (2 * c) * 2 * c
    assert sched.ktile_chunks * tt.KCHUNK == plan["tile"][2] // plan["tile"][3]
    # stride_eff + 1 stages in flight
    assert sched.inflight == plan["stride_eff"] + 1
    # ring depth: Eq.1 with the per-CTA overhead (task cache / barrier header / scratch), Eq.2 with the stage's pages
    spec = HardwareSpec(smem_max=tt.SMEM_MAX, page_size=tt.RING_PAGE,
                        instr_buf=tt.task_cache_bytes(CFG, 1, 148, sched.fuse_down), semaphores=tt.SMEM_RESERVED,
                        scratch=tt.scratch_bytes(CFG, sched, 1, 148))
    depth = compute_stage_count(compute_page_budget(spec, 1), 0, 0, 0, sched.stage_bytes // tt.RING_PAGE)
    assert sched.n_stage == depth == tt.ring_depth(CFG, sched) >= plan["n_stage"]
    assert plan["window"] == plan["n_stage"] * plan["per_stage"] <= plan["pages_required"]
    table = tt.build_task_table(CFG, sched)                    # and the schedule is executable
    assert table.header[4] == sched.n_stage and table.header[8] == sched.inflight
    ident = schedule_id(CFG)
    assert ident["content_hash"] == trace.content_hash and ident["program_order_checked"]
    assert order["fills"] == order["loader_ops"] > 0


def test_from_plan_rejects_inconsistent_or_oversized_plans():
    trace, knobs, _ = shipped_trace(CFG)
    plan = copy.deepcopy(trace.plan)
    plan["window"] += 1
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule.from_plan(plan, CFG, **knobs)
    plan = copy.deepcopy(trace.plan)
    plan["n_stage"] = 7
    plan["window"] = 7 * plan["per_stage"]
    plan["pages_required"] = plan["window"] + 1
    with pytest.raises(tt.ScheduleError):                       # seven 42 KB stages do not fit 227 KB
        tt.KernelSchedule.from_plan(plan, CFG, **knobs)
    plan = copy.deepcopy(trace.plan)
    plan["tile"][1] = 8                                         # fewer than two rows per consumer warp
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule.from_plan(plan, CFG, **knobs)


def test_program_order_check_rejects_hoists_across_stages():
    f = _files()
    trace, _, _ = shipped_trace(CFG)
    graph_text, hw_text = f["graph"].read_text(), f["hw"].read_text()
    assert check_program_order(trace, graph_text, hw_text)["consumer_stages"] > 10
    bad = copy.deepcopy(trace)
    prog = bad.plan["programs"]["Consumer"]
    # move the last MMA of the program to the front: work of the last stage ahead of the first
    prog.insert(0, prog.pop(len(prog) - 10))
    with pytest.raises(tt.ScheduleError):
        check_program_order(bad, graph_text, hw_text)
    bad = copy.deepcopy(trace)
    lp = bad.plan["programs"]["Loader"]
    lp[0], lp[5] = lp[5], lp[0]
    with pytest.raises(tt.ScheduleError):
        check_program_order(bad, graph_text, hw_text)


def test_models_without_a_trace_fall_back_to_the_profiled_default():
    from paper_2605_11581_b200.model_config import TINY

    assert shipped_trace(TINY) is None
    sched = default_schedule(TINY)
    assert sched.consumer_warps == 7 and sched.n_stage >= 3
    assert "profiled default" in schedule_id(TINY)["source"]


@pytest.mark.parametrize("name", SHIPPED[1:])
def test_larger_models_ship_traces_that_lower_to_the_profiled_schedule(name):
    """Qwen2.5-7B / Qwen3-8B: the searched plan lowers to the schedule profiling chose (42 x 512 tiles on seven warps,
    unfused down projection, ring depth from Eq.2), and a tensor-parallel rank never gets the fused down projection."""
    from paper_2605_11581_b200.schedules import PROFILED_DEFAULT, fit_schedule

    cfg = PRESETS[name]
    trace, knobs, order = shipped_trace(cfg)
    assert order is not None and order["fills"] > 0 and knobs["fuse_down"] is False
    sched = default_schedule(cfg)
    assert sched == fit_schedule(cfg, tt.KernelSchedule(n_stage=2, **PROFILED_DEFAULT))
    assert sched.inflight == trace.plan["stride_eff"] + 1
    assert schedule_id(cfg)["content_hash"] == trace.content_hash
    assert not default_schedule(cfg.shard(2), tp_size=2).fuse_down
