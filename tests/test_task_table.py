"""Host logic of the schedule -> device task table lowering (CPU only)."""

import re
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import QWEN25_1P5B, QWEN3_8B, TINY, TINY_QWEN3
from paper_2605_11581_b200.weights import random_weights

SCHED_TINY = tt.KernelSchedule(consumer_warps=8, n_stage=4, rows_per_tile=16, ktile_chunks=2, attn_min_chunk=8)


def test_split_rows_is_exact_cover_and_rotates():
    for n_units, n_sms, rot in [(2048, 148, 0), (1536, 148, 37), (10, 148, 140), (151936, 148, 5), (7, 3, 2)]:
        split = tt.split_rows(n_units, n_sms, rot)
        spans = sorted((f, c) for f, c in split if c)
        assert spans[0][0] == 0
        for (f0, c0), (f1, _) in zip(spans, spans[1:]):
            assert f0 + c0 == f1
        assert spans[-1][0] + spans[-1][1] == n_units
        counts = [c for _, c in split]
        assert max(counts) - min(counts) <= 1
        if n_units % n_sms:
            assert split[rot % n_sms][1] == n_units // n_sms + 1


@pytest.mark.parametrize("cfg", [TINY, TINY_QWEN3], ids=lambda c: c.name)
def test_packed_stream_covers_every_weight_exactly_once(cfg):
    """Pack, then invert the packing: every element of every matrix appears once."""
    table = tt.build_task_table(cfg, SCHED_TINY, n_sms=148)
    w = random_weights(cfg, seed=3)
    # replace weights by unique ids per matrix so the cover can be checked exactly
    packed = tt.pack_weights_reference(table, w)
    assert packed.nbytes == table.packed_weight_bytes
    perm = tt.chunk_permutation()
    seen = {}
    for task in table.tasks:
        ttype = int(task[tt.F_TYPE])
        if ttype not in tt.GEMV_TYPES:
            continue
        key_l = int(task[tt.F_LAYER])
        pos = int(task[tt.F_WOFF]) * 8
        k = int(task[tt.F_K])
        for tile, kt, rows, chunks in tt.stage_shapes(task):
            for r in range(rows):
                name, row = tt.virtual_row_source(cfg, ttype, int(task[tt.F_A]) + tile * int(task[tt.F_RT]) + r)
                cover = seen.setdefault((key_l if name != "lm_head" else -1, name), {})
                ks = cover.setdefault(row, np.zeros(k, dtype=np.int32))
                for c in range(chunks):
                    kidx = (kt * int(task[tt.F_KTC]) + c) * tt.KCHUNK + perm
                    valid = kidx < k
                    ks[kidx[valid]] += 1
                    src = (w.lm_head_matrix if name == "lm_head" else getattr(w.layers[key_l], name))
                    got = packed[pos:pos + tt.KCHUNK]
                    want = src[row].view(torch.int16).numpy().view(np.uint16)
                    assert (got[valid] == want[kidx[valid]]).all()
                    assert (got[~valid] == 0).all()
                    pos += tt.KCHUNK
    expect_rows = {"wq": cfg.q_dim, "wk": cfg.kv_dim, "wv": cfg.kv_dim, "wo": cfg.hidden,
                   "wgate": cfg.intermediate, "wup": cfg.intermediate, "wdown": cfg.hidden, "lm_head": cfg.vocab}
    assert len(seen) == 7 * cfg.n_layers + 1
    for (layer, name), cover in seen.items():
        assert len(cover) == expect_rows[name], (layer, name)
        for row, ks in cover.items():
            assert (ks == 1).all(), (layer, name, row)


def _n_active(table: tt.TaskTable, ctx: int) -> int:
    cl = max(table.sched.attn_min_chunk, -(-ctx // table.attn_chunks))
    cl = (cl + 7) & ~7
    return -(-ctx // cl)


def _simulate_dataflow(table: tt.TaskTable, ctx: int):
    """Replay the per-SM task lists against the kernel's data dependencies (tagged-word
    protocol, csrc/adamk.cu): a task can run once EVERY task that publishes one of the
    words it gathers has run (attention: every unit that is active at this context length;
    with a single active unit the unit publishes the merged output itself).  Returns the
    completion counts; raises on deadlock."""
    cfg = table.cfg
    n_active = _n_active(table, ctx)
    tasks = table.tasks
    L = cfg.n_layers

    def active(t):
        ty = int(t[tt.F_TYPE])
        if ty == tt.T_ATTN:
            return int(t[tt.F_B]) < n_active
        if ty == tt.T_MERGE:
            return n_active > 1
        return True

    total = {}
    for t in tasks:
        if active(t):
            key = (int(t[tt.F_LAYER]), int(t[tt.F_TYPE]))
            total[key] = total.get(key, 0) + 1
    done = {k: 0 for k in total}

    def complete(key):
        return done.get(key, 0) == total.get(key, 0)

    def ready(t) -> bool:
        ty, layer = int(t[tt.F_TYPE]), int(t[tt.F_LAYER])
        if ty == tt.T_LMHEAD:
            return complete((L - 1, tt.T_DOWN))
        if ty == tt.T_QKV:
            return layer == 0 or complete((layer - 1, tt.T_DOWN))
        if ty == tt.T_ATTN:
            return complete((layer, tt.T_QKV))
        if ty == tt.T_MERGE:
            return complete((layer, tt.T_ATTN))
        if ty == tt.T_OPROJ:   # gathers the merged attention output (+ the layer input as residual)
            return complete((layer, tt.T_ATTN)) and complete((layer, tt.T_MERGE))
        if ty == tt.T_GATEUP:
            return complete((layer, tt.T_OPROJ))
        if ty == tt.T_DOWN:
            return complete((layer, tt.T_GATEUP))
        raise AssertionError(ty)

    pc = table.sm_begin[:-1].astype(np.int64).copy()
    end = table.sm_begin[1:]
    while (pc < end).any():
        progressed = False
        for sm in range(table.n_sms):
            while pc[sm] < end[sm]:
                t = tasks[pc[sm]]
                if active(t):
                    if not ready(t):
                        break
                    done[(int(t[tt.F_LAYER]), int(t[tt.F_TYPE]))] += 1
                pc[sm] += 1
                progressed = True
        if not progressed:
            raise AssertionError(f"deadlock: pcs {pc[:8]}")
    return done


@pytest.mark.parametrize("ctx", [1, 8, 9, 100, 600])
def test_dataflow_has_no_deadlock(ctx):
    table = tt.build_task_table(TINY, SCHED_TINY, n_sms=148)
    done = _simulate_dataflow(table, ctx)
    assert done[(TINY.n_layers, tt.T_LMHEAD)] == table.header[12]
    n_active = _n_active(table, ctx)
    assert done[(0, tt.T_ATTN)] == TINY.n_q_heads * n_active
    assert done.get((0, tt.T_MERGE), 0) == (TINY.n_q_heads if n_active > 1 else 0)


def test_every_operator_covers_its_rows_exactly_once():
    """Per layer, the row ranges of each GEMV operator over all SMs tile [0, n_rows) exactly;
    attention units cover every (q head, chunk slot) once and every q head has one merge task."""
    for cfg, n_sms in ((TINY, 148), (TINY, 5), (QWEN25_1P5B, 148)):
        sched = SCHED_TINY if cfg is TINY else tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2)
        table = tt.build_task_table(cfg, sched, n_sms=n_sms)
        rows = {tt.T_QKV: cfg.qkv_rows, tt.T_OPROJ: cfg.hidden, tt.T_GATEUP: 2 * cfg.intermediate, tt.T_DOWN: cfg.hidden}
        t = table.tasks
        for layer in (0, cfg.n_layers - 1):
            for ty, n in rows.items():
                m = (t[:, tt.F_TYPE] == ty) & (t[:, tt.F_LAYER] == layer)
                spans = sorted((int(a), int(b)) for a, b in t[m][:, [tt.F_A, tt.F_B]])
                assert spans[0][0] == 0 and sum(b for _, b in spans) == n
                for (a0, b0), (a1, _) in zip(spans, spans[1:]):
                    assert a0 + b0 == a1
            m = (t[:, tt.F_TYPE] == tt.T_ATTN) & (t[:, tt.F_LAYER] == layer)
            units = {(int(a), int(b)) for a, b in t[m][:, [tt.F_A, tt.F_B]]}
            assert units == {(h, c) for h in range(cfg.n_q_heads) for c in range(table.attn_chunks)}
            m = (t[:, tt.F_TYPE] == tt.T_MERGE) & (t[:, tt.F_LAYER] == layer)
            assert sorted(int(a) for a in t[m][:, tt.F_A]) == list(range(cfg.n_q_heads))
        m = t[:, tt.F_TYPE] == tt.T_LMHEAD
        assert int(t[m][:, tt.F_B].sum()) == cfg.vocab


def test_warp_grid_geometry_is_executable():
    """Every GEMV task's warp grid satisfies the kernel's constraints (adamk_create re-checks them)."""
    for cfg, sched in ((QWEN25_1P5B, tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2)),
                       (QWEN25_1P5B, tt.KernelSchedule(consumer_warps=8, n_stage=5, rows_per_tile=64, ktile_chunks=1)),
                       (QWEN3_8B, tt.KernelSchedule(consumer_warps=4, n_stage=3, rows_per_tile=32, ktile_chunks=3)),
                       (TINY, SCHED_TINY)):
        table = tt.build_task_table(cfg, sched, n_sms=148)
        for task in table.tasks:
            if int(task[tt.F_TYPE]) not in tt.GEMV_TYPES:
                continue
            wr, wk, rw = tt.unpack_geom(int(task[tt.F_GEOM]))
            assert wr * wk == sched.consumer_warps and 1 <= rw <= tt.MAX_RW
            assert int(task[tt.F_RT]) == wr * rw
            assert wk == 1 or int(task[tt.F_RT]) <= 32
            assert wk & (wk - 1) == 0                      # K groups are a power of two (shift / mask in the kernel)
            assert int(task[tt.F_RT]) * int(task[tt.F_KTC]) * 512 <= sched.stage_bytes
            assert int(task[tt.F_NTILES]) == -(-int(task[tt.F_B]) // int(task[tt.F_RT]))
            assert int(task[tt.F_NKTILES]) == -(-int(task[tt.F_KCHUNKS]) // int(task[tt.F_KTC]))
            if int(task[tt.F_TYPE]) == tt.T_GATEUP:
                assert rw % 2 == 0 and int(task[tt.F_A]) % 2 == 0 and int(task[tt.F_B]) % 2 == 0
            # rows a warp group may touch past the tile end stay inside the ring slot
            assert wr * rw * int(task[tt.F_KTC]) * 512 <= sched.stage_bytes


def test_dataflow_full_model_and_small_gpu():
    sched = tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2)
    table = tt.build_task_table(QWEN25_1P5B, sched, n_sms=148)
    _simulate_dataflow(table, 513)
    s = table.summary()
    assert s["packed_weight_bytes"] * 1.0 <= QWEN25_1P5B.weight_bytes_per_token()
    assert s["stream_bytes_max"] - s["stream_bytes_min"] <= 64 * 1024
    assert int(np.diff(table.sm_begin).max()) * 32 <= tt.task_cache_bytes(QWEN25_1P5B)
    small = tt.build_task_table(TINY, SCHED_TINY, n_sms=5)
    _simulate_dataflow(small, 33)
    assert int(np.diff(small.sm_begin).max()) * 32 <= tt.task_cache_bytes(TINY, n_sms=5)


def test_schedule_validation():
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(consumer_warps=8, rows_per_tile=8)          # one row per warp splits gate/up pairs
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(consumer_warps=6)
    with pytest.raises(tt.ScheduleError):
        tt.build_task_table(QWEN25_1P5B, tt.KernelSchedule(n_stage=16, ktile_chunks=1))   # 16 x 32 KB > 227 KB
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(n_stage=3, inflight=4)
    s = tt.KernelSchedule.from_plan({"tile": [16, 32, 1024, 2], "n_stage": 5, "consumer_warps": 16})
    assert (s.rows_per_tile, s.ktile_chunks, s.stage_bytes) == (32, 2, 32768)
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule.from_plan({"tile": [16, 16, 64, 1], "n_stage": 2, "consumer_warps": 8})


def test_blob_layout_matches_header():
    table = tt.build_task_table(TINY, SCHED_TINY, n_sms=148)
    raw = np.frombuffer(table.blob, dtype="<i4")
    assert raw[0] == tt.MAGIC and raw[1] == tt.VERSION and raw[2] == 148
    assert raw.size == tt.HEADER_INTS + 149 + raw[6] * tt.TASK_INTS
    assert tt.max_stages_that_fit(QWEN3_8B, tt.KernelSchedule(ktile_chunks=1)) >= 4


def test_cabi_exports_every_declared_symbol():
    """The C-ABI library loads and exports everything include/adamk.h declares
    (no compute calls: there is no GPU here)."""
    from paper_2605_11581_b200 import build, plugin

    build.build()
    header = (Path(__file__).resolve().parents[1] / "include" / "adamk.h").read_text()
    declared = set(re.findall(r"\b(adamk_[a-z0-9_]+)\s*\(", header))
    declared -= {"adamk_handle", "adamk_stream"}
    assert declared == set(plugin.EXPORTS)
    lib = plugin.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.adamk_abi_version() == plugin.ABI_VERSION


def test_cabi_exports_prefill_operators():
    """include/adamk_prefill.h: the Prefill operators live in the same library and every declared symbol is exported."""
    from paper_2605_11581_b200 import build, plugin, prefill

    build.build()
    header = (Path(__file__).resolve().parents[1] / "include" / "adamk_prefill.h").read_text()
    declared = set(re.findall(r"\b(adamk_(?:prefill|batch)(?:_[a-z_]+)?)\s*\(", header))
    assert declared == set(prefill.PREFILL_EXPORTS)
    lib = plugin.load_library()
    for name in declared:
        assert hasattr(lib, name), name


def test_prefill_gate_up_interleave():
    """Host-side weight layout of the fused SwiGLU GEMM: blocks of gate rows followed by the up rows of the same
    features, zero rows padding the intermediate size to a whole block."""
    import torch

    from paper_2605_11581_b200.prefill import interleave_gate_up

    g = torch.arange(6 * 4, dtype=torch.float32).reshape(6, 4)
    u = -g
    w = interleave_gate_up(g, u, block=4)
    assert w.shape == (16, 4)
    assert torch.equal(w[0:4], g[0:4]) and torch.equal(w[4:8], u[0:4])
    assert torch.equal(w[8:10], g[4:6]) and torch.equal(w[12:14], u[4:6])
    assert w[10:12].abs().sum() == 0 and w[14:16].abs().sum() == 0


def test_search_to_schedule_to_task_table():
    """Offline half -> online half: the planner's search on the share of a layer one SM executes
    (mkplan.model_graph.build_sm_slice_graph) yields a SolidifiedTrace whose plan lowers to a kernel schedule
    and a task table (the flow of PAPER.md:195-197: search, solidify, replay)."""
    import json
    from pathlib import Path

    from paper_2605_11581_b200.mkplan import model_graph, search

    cfg = TINY
    graph = model_graph.build_sm_slice_graph(cfg, 64, n_sms=148)
    ops = {o["id"]: o["dims"] for o in graph["operators"]}
    assert ops["qkv"]["n"] == -(-cfg.qkv_rows // 148) and ops["qkv"]["k"] == cfg.hidden
    assert ops["upgate"]["n"] == 2 * -(-cfg.intermediate // 148) and ops["down"]["k"] == cfg.intermediate
    hw = (Path(tt.__file__).parent / "mkplan" / "fixtures" / "b200.json").read_text()
    space = {"block_m": [16], "block_n": [16, 32], "block_k": [256], "k_split": [1], "consumer_warps": [4, 8],
             "n_stage": [2, 3], "prefetch_stride": [1], "swizzles": [31]}
    trace = search.run_search(json.dumps(graph), hw, json.dumps(space), 100)
    again = search.parse_trace(search.serialize_trace(trace))
    assert again.plan == trace.plan
    sched = tt.KernelSchedule.from_plan(trace.plan, attn_min_chunk=16)
    assert sched.consumer_warps == trace.plan["consumer_warps"] and sched.n_stage == trace.plan["n_stage"]
    assert sched.rows_per_tile <= tt.MAX_RW * sched.consumer_warps and sched.ktile_chunks == 1
    table = tt.build_task_table(cfg, sched, n_sms=148)
    _simulate_dataflow(table, 40)
    # a plan tile taller than eight rows per warp is split into several kernel tiles
    tall = tt.KernelSchedule.from_plan({"tile": [16, 64, 512, 2], "n_stage": 3, "consumer_warps": 4})
    assert (tall.rows_per_tile, tall.ktile_chunks) == (32, 1)


def test_prefill_pass_entry_validates_on_the_host():
    """`adamk_prefill` (the whole Prefill pass behind one C call): workspace sizing and argument checks are host
    arithmetic and need no GPU."""
    import ctypes as C

    from paper_2605_11581_b200 import prefill

    lib = prefill._lib()
    cfg = QWEN25_1P5B
    i_pad = -(-cfg.intermediate // 128) * 128
    model = prefill._PassModel(cfg.n_layers, cfg.hidden, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, i_pad, 4096, cfg.rms_eps,
                               cfg.n_kv_heads * 4096 * cfg.head_dim * 2)
    T, P = 512, 1
    need = lib.adamk_prefill_workspace_bytes(C.byref(model), T, 0, P)
    lower = 2 * T * (cfg.hidden + cfg.q_dim + cfg.q_dim + i_pad) + 4 * T * cfg.qkv_rows + 2 * cfg.kv_dim * 512
    assert lower <= need <= lower + 6 * 256
    assert lib.adamk_prefill_workspace_bytes(C.byref(model), T, 0, 2) > need
    assert lib.adamk_prefill_workspace_bytes(C.byref(model), 0, 0, 1) == 0          # no tokens
    assert lib.adamk_prefill_workspace_bytes(C.byref(model), T, 0, 3) == 0          # planes must be 1 or 2
    bad = prefill._PassModel(cfg.n_layers, cfg.hidden, cfg.n_q_heads, cfg.n_kv_heads, 96, i_pad, 4096, cfg.rms_eps, 1)
    assert lib.adamk_prefill_workspace_bytes(C.byref(bad), T, 0, 1) == 0            # head_dim 64 / 128 only
    layers = (prefill._PassLayer * cfg.n_layers)()
    rc = lib.adamk_prefill(C.byref(model), layers, None, None, None, None, T, 0, P, None, None, None, None, None)
    assert rc != 0 and b"NULL argument" in lib.adamk_prefill_pass_last_error()
    one = C.c_void_p(256)
    rc = lib.adamk_prefill(C.byref(model), layers, one, one, one, one, 4096, 1, P, one, one, one, one, None)
    assert rc != 0 and b"does not fit the KV cache" in lib.adamk_prefill_pass_last_error()
