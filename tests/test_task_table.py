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


PHASE_OF = {tt.T_QKV: 0, tt.T_ATTN: 1, tt.T_OPROJ: 2, tt.T_GATEUP: 3, tt.T_DOWN: 4}


def _simulate_dataflow(table: tt.TaskTable, ctx: int):
    """Replay the per-SM task lists against the kernel's data dependencies (tagged-word
    protocol): a task needs EVERY task of the previous phase to have published its
    outputs (attention: every unit that is active at this context length).  Returns the
    number of rounds; raises on deadlock."""
    cfg, sched = table.cfg, table.sched
    cl = max(sched.attn_min_chunk, -(-ctx // table.attn_chunks))
    cl = (cl + 7) & ~7
    n_active = -(-ctx // cl)
    tasks = table.tasks
    L = cfg.n_layers

    def active(t):
        return int(t[tt.F_TYPE]) != tt.T_ATTN or int(t[tt.F_B]) < n_active

    total = {}
    for t in tasks:
        if active(t):
            key = (int(t[tt.F_LAYER]), int(t[tt.F_TYPE]))
            total[key] = total.get(key, 0) + 1
    done = {k: 0 for k in total}

    def ready(t) -> bool:
        ty, layer = int(t[tt.F_TYPE]), int(t[tt.F_LAYER])
        if ty == tt.T_LMHEAD:
            prev = (L - 1, tt.T_DOWN)
        elif ty == tt.T_QKV:
            if layer == 0:
                return True
            prev = (layer - 1, tt.T_DOWN)
        else:
            prev = (layer, {tt.T_ATTN: tt.T_QKV, tt.T_OPROJ: tt.T_ATTN, tt.T_GATEUP: tt.T_OPROJ,
                            tt.T_DOWN: tt.T_GATEUP}[ty])
        return done[prev] == total[prev]

    pc = table.sm_begin[:-1].astype(np.int64).copy()
    end = table.sm_begin[1:]
    rounds = 0
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
        rounds += 1
        if not progressed:
            raise AssertionError(f"deadlock: pcs {pc[:8]}")
    return rounds, done


@pytest.mark.parametrize("ctx", [1, 8, 9, 100, 600])
def test_dataflow_has_no_deadlock(ctx):
    table = tt.build_task_table(TINY, SCHED_TINY, n_sms=148)
    _, done = _simulate_dataflow(table, ctx)
    assert done[(TINY.n_layers, tt.T_LMHEAD)] == table.header[12]


def test_every_sm_updates_the_residual_stream():
    """The residual stream is replicated per CTA and brought up to date by the QKV, gate/up and
    LM-head prologues: every SM must own exactly one of each per layer, even with zero rows."""
    for n_sms in (148, 5, 300):
        table = tt.build_task_table(TINY, SCHED_TINY, n_sms=n_sms)
        for sm in range(n_sms):
            ts = table.tasks_of(sm)
            for layer in range(TINY.n_layers):
                for ty in (tt.T_QKV, tt.T_GATEUP):
                    assert ((ts[:, tt.F_TYPE] == ty) & (ts[:, tt.F_LAYER] == layer)).sum() == 1
            assert (ts[:, tt.F_TYPE] == tt.T_LMHEAD).sum() == 1


def test_dataflow_full_model_and_small_gpu():
    sched = tt.KernelSchedule(consumer_warps=8, n_stage=5, rows_per_tile=16, ktile_chunks=3)
    table = tt.build_task_table(QWEN25_1P5B, sched, n_sms=148)
    _simulate_dataflow(table, 513)
    s = table.summary()
    assert s["packed_weight_bytes"] * 1.0 <= QWEN25_1P5B.weight_bytes_per_token()
    assert s["stream_bytes_max"] - s["stream_bytes_min"] <= 64 * 1024
    small = tt.build_task_table(TINY, SCHED_TINY, n_sms=5)
    _simulate_dataflow(small, 33)


def test_schedule_validation():
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(consumer_warps=8, rows_per_tile=8)          # one row per warp splits gate/up pairs
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(consumer_warps=6)
    with pytest.raises(tt.ScheduleError):
        tt.build_task_table(QWEN25_1P5B, tt.KernelSchedule(n_stage=16, ktile_chunks=4))   # 16 x 32 KB > 227 KB
    s = tt.KernelSchedule.from_plan({"tile": [16, 32, 1024, 2], "n_stage": 5, "consumer_warps": 16})
    assert (s.rows_per_tile, s.ktile_chunks, s.stage_bytes) == (32, 2, 32768)
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule.from_plan({"tile": [16, 16, 64, 1], "n_stage": 2, "consumer_warps": 8})


def test_blob_layout_matches_header():
    table = tt.build_task_table(TINY, SCHED_TINY, n_sms=148)
    raw = np.frombuffer(table.blob, dtype="<i4")
    assert raw[0] == tt.MAGIC and raw[1] == tt.VERSION and raw[2] == 148
    assert raw.size == tt.HEADER_INTS + 149 + raw[6] * tt.TASK_INTS
    assert tt.max_stages_that_fit(QWEN3_8B, tt.KernelSchedule(ktile_chunks=4)) >= 4


def test_cabi_exports_every_declared_symbol():
    """The C-ABI library loads and exports everything include/adamk.h declares
    (no compute calls: there is no GPU here)."""
    from paper_2605_11581_b200 import build, plugin

    build.build()
    header = (Path(__file__).resolve().parents[1] / "include" / "adamk.h").read_text()
    declared = set(re.findall(r"\b(adamk_[a-z_]+)\s*\(", header))
    declared -= {"adamk_handle", "adamk_stream"}
    assert declared == set(plugin.EXPORTS)
    lib = plugin.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.adamk_abi_version() == plugin.ABI_VERSION
