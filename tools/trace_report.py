#!/usr/bin/env python
"""Per-task timeline of one decode step (in-kernel %globaltimer stamps) -> phase table.

    python tools/trace_report.py qwen2.5-1.5b 512 key=value ... (KernelSchedule fields)

Stamps per task: 0 start, 1 inputs gathered (attention: q prepared), 2 body done (GEMV), 3 K/V blocks
done (attention), 7 end.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.weights import random_weights


def collect(name, ctx0, kw, steps=3):
    cfg = PRESETS[name]
    w = random_weights(cfg, 0, device="cuda")
    plug = MegaKernelPlugin(cfg, tt.KernelSchedule(**kw), max_ctx=ctx0 + 64)
    plug.bind_weights(w)
    kc, vc = plug.kv_view(); kc.normal_(); vc.normal_()
    plug.set_state(1, ctx0)
    for _ in range(3):
        plug.enqueue()
    plug.check()
    tr = plug.enable_trace(True)
    out = []
    for _ in range(steps):
        tr.zero_()
        plug.set_state(1, ctx0)
        plug.enqueue()
        plug.check()
        out.append(tr.cpu().numpy().copy())
    return plug, out


def report(plug, tr):
    tasks = plug.table.tasks
    types, layers = tasks[:, tt.F_TYPE], tasks[:, tt.F_LAYER]
    ran = tr[:, 7] > 0
    t0 = tr[ran][:, 0].min()
    rel = (tr.astype(np.float64) - float(t0)) / 1e3  # us
    L = plug.cfg.n_layers
    order = [tt.T_QKV, tt.T_ATTN, tt.T_MERGE, tt.T_OPROJ, tt.T_GATEUP, tt.T_DOWN, tt.T_DOWNK, tt.T_HRED]
    print(f"step total (first stamp -> last end): {rel[ran][:, 7].max():.1f} us")
    acc = {}
    prev_end = 0.0
    for layer in range(L + 1):
        for ty in (order if layer < L else [tt.T_LMHEAD]):
            m = ran & (types == ty) & (layers == layer)
            if not m.any():
                continue
            r = rel[m]
            gathered = r[:, 1] if ty not in (tt.T_MERGE, tt.T_DOWNK) else r[:, 0]
            end = r[:, 7]
            d = dict(phase=end.max() - prev_end,                 # critical-path length of the op
                     first_in=gathered.min() - prev_end,         # first SM has its inputs after the previous op ended
                     last_in=gathered.max() - prev_end,
                     body_mean=(end - gathered).mean(), body_max=(end - gathered).max(),
                     end_spread=end.max() - end.min(), early=(prev_end - r[:, 0]).mean())
            if ty == tt.T_ATTN:
                d.update(a_kv=(r[:, 4] - r[:, 1]).mean(), a_blocks=(r[:, 3] - r[:, 4]).mean(),
                         a_comb=(r[:, 5] - r[:, 3]).mean(), a_out=(r[:, 7] - r[:, 5]).mean(), a_qprep=(r[:, 1] - r[:, 0]).mean())
            prev_end = end.max()
            if layer in (0,):
                continue  # cold start excluded from the means
            a = acc.setdefault(tt.TYPE_NAMES[ty], [])
            a.append(d)
    print(f"{'op':8s} {'phase':>7s} {'first_in':>9s} {'last_in':>8s} {'body':>7s} {'bodymax':>8s} {'endsprd':>8s} {'waiting':>8s}   (us, mean over layers >= 1)")
    tot = 0.0
    for op, a in acc.items():
        mean = {k: float(np.mean([d[k] for d in a])) for k in a[0]}
        if op != "lmhead":
            tot += mean["phase"]
        print(f"{op:8s} {mean['phase']:7.2f} {mean['first_in']:9.2f} {mean['last_in']:8.2f} {mean['body_mean']:7.2f} "
              f"{mean['body_max']:8.2f} {mean['end_spread']:8.2f} {mean['early']:8.2f}   (x{len(a)})")
        if op == "attn":
            print("   attn unit: start->q ready %.2f | ->K/V landed %.2f | blocks %.2f | warp merge sync %.2f | records out %.2f" % tuple(
                mean[k] for k in ("a_qprep", "a_kv", "a_blocks", "a_comb", "a_out")))
    print(f"mean per-layer time {tot:.2f} us")


if __name__ == "__main__":
    name, ctx0 = sys.argv[1], int(sys.argv[2])
    kw = {}
    for a in sys.argv[3:]:
        k, v = a.split("=")
        kw[k] = int(v)
    plug, traces = collect(name, ctx0, kw)
    report(plug, traces[-1])
