#!/usr/bin/env python
"""Soak test of the decode MegaKernel: N free-running greedy steps (device-resident loop), twice, from the same state.
Checks that no step trips the in-kernel watchdog (a lost tagged word or a stalled ring would), that the two runs emit
identical token streams (fixed summation order), and reports the step-time distribution over windows of 1000 steps.

    python tools/soak.py [model] [steps] [ctx0]
"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.schedules import default_schedule
from paper_2605_11581_b200.weights import random_weights

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
ctx0 = int(sys.argv[3]) if len(sys.argv) > 3 else 64
cfg = PRESETS[name]
w = random_weights(cfg, 0, device="cuda")
plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=ctx0 + steps + 8)
plug.bind_weights(w)
kc, vc = plug.kv_view()
g = torch.Generator(device="cuda").manual_seed(1)
k0 = torch.randn(kc[:, :, :, :ctx0].shape, device="cuda", generator=g).to(kc.dtype)
v0 = torch.randn(vc[:, :, :, :ctx0].shape, device="cuda", generator=g).to(vc.dtype)
streams, windows = [], []
for run in range(2):
    kc.zero_(); vc.zero_()
    kc[:, :, :, :ctx0] = k0; vc[:, :, :, :ctx0] = v0
    plug.set_state(17, ctx0)
    toks = torch.empty(steps, dtype=torch.int32, device="cuda")
    t_run = time.time()
    for s0 in range(0, steps, 1000):
        n = min(1000, steps - s0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            plug.enqueue()
            toks[s0 + i:s0 + i + 1].copy_(plug.next_token, non_blocking=True)
        e1.record()
        plug.check()                                   # raises on a watchdog report
        windows.append((run, s0 + ctx0, e0.elapsed_time(e1) / n * 1e3))
    streams.append(toks.cpu())
    print(f"run {run}: {steps} steps in {time.time() - t_run:.1f} s, context {ctx0} -> {ctx0 + steps}, no device error", flush=True)
same = bool((streams[0] == streams[1]).all())
print(f"token streams identical: {same}; distinct tokens {len(set(streams[0].tolist()))}")
for run, ctx, us in windows[:: max(1, len(windows) // 12)]:
    print(f"  run {run} context {ctx:6d}: {us:7.1f} us/step")
assert same
