#!/usr/bin/env python
"""Per-task timeline of one decode step (in-kernel %globaltimer stamps) -> phase table.

    python tools/trace_report.py qwen2.5-1.5b 512 8 5 16 4 [out.json]
"""
import json
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
        plug.enqueue()
        plug.check()
        out.append(tr.cpu().numpy().copy())
    return plug, out


def report(plug, tr):
    tasks = plug.table.tasks
    types, layers = tasks[:, tt.F_TYPE], tasks[:, tt.F_LAYER]
    ran = tr[:, 7] > 0
    t0 = tr[ran][:, 0].min()
    rel = (tr - t0) / 1e3  # us
    L = plug.cfg.n_layers
    order = [tt.T_QKV, tt.T_ATTN, tt.T_OPROJ, tt.T_GATEUP, tt.T_DOWN]
    rows = []
    prev_end = 0.0
    for layer in range(L + 1):
        for ty in (order if layer < L else [tt.T_LMHEAD]):
            m = ran & (types == ty) & (layers == layer)
            if not m.any():
                continue
            r = rel[m]
            rows.append(dict(layer=layer, op=tt.TYPE_NAMES[ty], n=int(m.sum()),
                             first_dep=float(r[:, 1].min()), last_dep=float(r[:, 1].max()),
                             last_pro=float(r[:, 2].max()), first_end=float(r[:, 7].min()),
                             last_end=float(r[:, 7].max()), prev_end=prev_end,
                             wait_mean=float((r[:, 1] - r[:, 0]).mean()), pro_mean=float((r[:, 2] - r[:, 1]).mean()),
                             body_mean=float((r[:, 7] - r[:, 2]).mean()), body_max=float((r[:, 7] - r[:, 2]).max()),
                             seg=[float(np.mean(r[:, k] - r[:, 1])) if (tr[m][:, k] > 0).all() else float('nan') for k in range(2, 8)]))
            prev_end = rows[-1]["last_end"]
    total = prev_end
    print(f"step total (first stamp -> last end): {total:.1f} us")
    print(f"{'op':8s} {'phase':>8s} {'sync':>7s} {'dep spread':>10s} {'prologue':>8s} {'body mean':>9s} {'body max':>8s} {'end spread':>10s}")
    agg = {}
    for r in rows:
        a = agg.setdefault(r["op"], [])
        a.append([r["last_end"] - r["prev_end"], r["first_dep"] - r["prev_end"], r["last_dep"] - r["first_dep"],
                  r["pro_mean"], r["body_mean"], r["body_max"], r["last_end"] - r["first_end"]])
    for op, a in agg.items():
        a = np.array(a)
        if len(a) > 2:
            a = a[1:]  # drop layer 0 (cold start)
        m = a.mean(0)
        print(f"{op:8s} {m[0]:8.2f} {m[1]:7.2f} {m[2]:10.2f} {m[3]:8.2f} {m[4]:9.2f} {m[5]:8.2f} {m[6]:10.2f}   (x{len(a)})")
    segs = {}
    for r in rows:
        segs.setdefault(r["op"], []).append(r["seg"])
    print("mean time of stamps 2..7 after the dependency was met (us; attn: 2 q-prep, 5 K landed, 3 scores, 6 V landed, 4 PV, 7 end):")
    for op, a in segs.items():
        a = np.array(a)
        if len(a) > 2:
            a = a[1:]
        print(f"  {op:8s}", " ".join(f"{v:6.2f}" for v in np.nanmean(a, axis=0)))
    per_layer = sum(np.array(a)[1:].mean(0)[0] for op, a in agg.items() if op != "lmhead" and len(a) > 2)
    print(f"mean per-layer time {per_layer:.2f} us; lm head phase {np.array(agg['lmhead'])[:, 0].mean():.1f} us")
    return rows


if __name__ == "__main__":
    name, ctx0 = sys.argv[1], int(sys.argv[2])
    kw = dict(consumer_warps=int(sys.argv[3]), n_stage=int(sys.argv[4]), rows_per_tile=int(sys.argv[5]),
              ktile_chunks=int(sys.argv[6]))
    plug, traces = collect(name, ctx0, kw)
    rows = report(plug, traces[-1])
    if len(sys.argv) > 7:
        Path(sys.argv[7]).write_text(json.dumps(rows))
