#!/usr/bin/env python
"""Benchmark of the decode MegaKernel hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one decode step (one token) of BASELINE.json configs[1]:
Qwen2.5-1.5B, random-init bf16, batch 1, after a 512-token prompt; K steps are
timed after W warm-up steps (defaults 128 / 16).  One JSON line is printed by
rank 0:

  value      whole-job decode tokens/s with token/position state resident in HBM
             (steps enqueued back to back, CUDA events on the launching stream)
  e2e        the same metric through the host-facing plugin call: per step the
             token + position are copied from pinned host memory, the step runs,
             and the next token is read back to the host
  roofline   weight-streaming HBM roofline of the (single) kernel: algorithmic
             bytes per launch / mean launch time vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the CPU oracle (oracle/decode_ref.py, kind "port": the reference
             ships no numeric decode path) timed on this box's host cores on a
             bounded sample of the same workload

`--impl reference` times that CPU oracle as the reference arm (same metric and
config).  N > 1 runs N independent replicas (config #2 has 2 KV heads and does
not shard past TP=2: "replicas only"), one rank per GPU.  With
`--tp` (BASELINE.json configs[3]: `--model qwen3-8b --tp --gpus N`) the N ranks
are tensor-parallel shards of ONE sequence instead: every rank launches one
kernel per token and the kernels exchange their partial rows through
peer-mapped workspaces (no NCCL on the data path); `value` is then the
sequence's tokens/s and `scaling` is "strong".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch

from paper_2605_11581_b200.model_config import get_config
from paper_2605_11581_b200.schedules import default_schedule, schedule_id
from paper_2605_11581_b200.weights import random_weights, rope_table

METRIC = "decode_tokens_per_s"
UNIT = "tokens/s"
PROMPT_LEN = 512


def measured_peak() -> tuple[float, str]:
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        return float(json.loads(path.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock / throttle-reason sampling during the timed region: NVML from a thread (first sample taken
    synchronously, so a short region is never left without one), `nvidia-smi -lms` as the fallback."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.sm, self.mx, self.flags, self._stop, self._thread, self._nvml = [], None, set(), False, None, None

    def _sample_nvml(self):
        nv, h = self._nvml
        self.sm.append(int(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons")
                else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
        for name, bit in (("hw_slowdown", 0x8), ("sw_power_cap", 0x4), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40)):
            if r & bit:
                self.flags.add(name)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            # CUDA_VISIBLE_DEVICES may renumber the devices: address the GPU by the UUID torch reports
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            try:
                h = nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml = (nv, h)
            self.mx = int(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._sample_nvml()

            def loop():
                while not self._stop:
                    try:
                        self._sample_nvml()
                    except Exception:
                        break
                    time.sleep(0.02)

            self._thread = threading.Thread(target=loop, daemon=True)
            self._thread.start()
            return
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self._nvml is not None:
            try:
                self._sample_nvml()              # one more, still under load
            except Exception:
                pass
            self._stop = True
            if self._thread is not None:
                self._thread.join(timeout=1.0)
            sm = sorted(self.sm)
            return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.mx, "reasons": sorted(self.flags),
                    "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm = sorted(int(r[0]) for r in self.rows if r and r[0].isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) >= 6 for n, v in zip(names, r[2:6]) if v.startswith("Active")})
        mx = [int(r[1]) for r in self.rows if len(r) > 1 and r[1].isdigit()]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": "nvidia-smi"}


def cpu_decode_sample(cfg, weights, prompt, n_steps: int, warmup: int = 2) -> dict:
    """Time the CPU oracle on a bounded sample: prefill the prompt, then n decode steps."""
    from oracle.decode_ref import RefDecoder

    torch.set_num_threads(os.cpu_count() or 1)
    cos, sin = rope_table(cfg, len(prompt) + n_steps + warmup + 8)
    dec = RefDecoder(cfg, weights, len(prompt) + n_steps + warmup + 8, cos, sin)
    logits = dec.prefill(prompt)
    tok, pos = int(torch.argmax(logits)), len(prompt)
    for _ in range(warmup):
        tok = int(torch.argmax(dec.step([tok], [pos])[0]))
        pos += 1
    t0 = time.perf_counter()
    for _ in range(n_steps):
        tok = int(torch.argmax(dec.step([tok], [pos])[0]))
        pos += 1
    dt = time.perf_counter() - t0
    return {"value": n_steps / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{n_steps} greedy decode steps after a {len(prompt)}-token prompt, fp32 compute on the same "
                      f"bf16 weights, torch CPU ({torch.get_num_threads()} threads)", "ms_per_step": dt / n_steps * 1e3}


def base_line(args, cfg, n_gpus: int) -> dict:
    return {"metric": METRIC, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, random prompt ids; no network for checkpoints)",
            "config": {"workload": f"{cfg.name} batch-1 greedy decode after a {PROMPT_LEN}-token prompt "
                                   f"(BASELINE.json configs[{1 if cfg.name == 'qwen2.5-1.5b' else 3}])",
                       "model": cfg.name, "batch": 1,
                       "prompt_len": PROMPT_LEN, "parallelism": "replicas" if n_gpus > 1 else "single",
                       "l2_policy": f"inputs larger than L2: every step streams the "
                                    f"{cfg.weight_bytes_per_token() / 1e9:.2f} GB weight set",
                       # the solidified schedule the workload is decoded with (mkplan search output; both arms name it so
                       # that their config objects are identical -- the CPU arm itself has no schedule)
                       "schedule": schedule_id(cfg)}}


def run_reference(args) -> None:
    """Reference arm: the CPU oracle on the host cores (the reference has no numeric decode)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = get_config(args.model)
    w = random_weights(cfg, seed=0)
    g = torch.Generator().manual_seed(1)
    prompt = torch.randint(0, cfg.vocab, (PROMPT_LEN,), generator=g).tolist()
    res = cpu_decode_sample(cfg, w, prompt, n_steps=args.steps, warmup=args.warmup)
    line = base_line(args, cfg, args.gpus)
    line.update({"impl": "reference", "value": res["value"], "ms_per_step": res["ms_per_step"],
                 "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
                 "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "gpu_launches": 0, "dtype": "f32 compute on bf16 weights"})
    print(json.dumps(line))


def prefill_sample(cfg, w, dev, local: int, tokens: int = 4096, iters: int = 5) -> dict:
    """Extra, outside the timed decode region: the Prefill half of the hybrid engine on the
    hand-written tcgen05 GEMM (paper_2605_11581_b200/prefill.py), 4096 prompt tokens, against the tensor roofline
    (MEASURED_PEAKS.json sustained bf16 TFLOP/s).  GEMM FLOPs only: 2 x tokens x layer weight elements x planes."""
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.prefill import TensorCorePrefill

    plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=tokens + 16, device=local)
    plug.bind_weights(w)
    toks = torch.randint(0, cfg.vocab, (tokens,), generator=torch.Generator().manual_seed(2)).to(dev)
    peak = None
    pfile = ROOT / "MEASURED_PEAKS.json"
    if pfile.exists():
        peak = json.loads(pfile.read_text()).get("bf16_tflops_sustained")
    out = {"tokens": tokens, "attention": "own tcgen05 flash kernel (csrc/prefill_attn.cu, bf16 Q/K/V/P, fp32 scores and output)", "peak_tflops": peak, "peak_kind": "measured sustained cuBLAS bf16"}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for planes in (1, 2):
        pre = TensorCorePrefill(cfg, w, plug, planes=planes, attention="bf16")
        for _ in range(3):
            pre.run(toks)
        torch.cuda.synchronize(dev)
        n0 = pre.launches
        e0.record()
        for _ in range(iters):
            pre.run(toks)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / iters
        mats = cfg.qkv_rows * cfg.hidden + cfg.hidden * cfg.q_dim + 3 * cfg.intermediate * cfg.hidden
        flops = 2.0 * tokens * mats * cfg.n_layers * planes
        # + causal attention (QK^T and PV, half of the square), one plane
        flops += 4.0 * cfg.n_q_heads * cfg.head_dim * tokens * tokens / 2 * cfg.n_layers
        out[f"planes{planes}"] = {"ms": ms, "tokens_per_s": tokens * 1e3 / ms, "tflops": flops / ms / 1e9,
                                  "frac_of_peak": None if not peak else flops / ms / 1e9 / peak,
                                  "own_kernel_launches": (pre.launches - n0) // iters}
        del pre
    plug.close()
    return out


def batch_decode_sample(cfg, w, dev, local: int, ctx: int = 2048, steps: int = 32) -> dict:
    """Extra, outside the timed batch-1 region: BASELINE.json configs[2], batched decode on the tensor cores
    (paper_2605_11581_b200/batch_decode.py): one CUDA-graph launch per step of B sequences, every sequence at context
    ``ctx``.  `weights_gbs` = the model's weight bytes / step time (the weights are streamed once per step)."""
    from paper_2605_11581_b200.batch_decode import BatchedDecoder

    out = {"context": ctx, "steps": steps, "launch": "one CUDA graph of 10 kernels per layer"}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for B in (8, 64):
        dec = BatchedDecoder(cfg, w, B, ctx + steps + 32, device=local)
        g = torch.Generator().manual_seed(3)
        dec.set_state(torch.randint(0, cfg.vocab, (B,), generator=g).tolist(), [ctx] * B)
        dec.capture()
        for _ in range(8):
            dec.step()
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(steps):
            dec.step()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / steps
        out[f"batch{B}"] = {"ms_per_step": ms, "tokens_per_s": B * 1e3 / ms, "own_kernel_launches_per_step": dec.launches_per_step,
                            "weights_gbs": cfg.weight_bytes_per_token() / ms / 1e6}
        del dec
        torch.cuda.empty_cache()
    return out


def run_ours(args) -> None:
    from paper_2605_11581_b200.plugin import MegaKernelPlugin

    from paper_2605_11581_b200.dist_utils import RankGroup

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = RankGroup()            # nccl when WORLD_SIZE > 1; N replicas, no data-path collective
    rank, world, dist = group.rank, group.world, group.dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    full_cfg = get_config(args.model)
    tp = world if (args.tp and world > 1) else 1
    cfg = full_cfg.shard(tp)                      # this rank's dimensions (the whole model when tp == 1)
    w = random_weights(full_cfg, seed=0, device=dev).shard(rank, tp)   # same seed on every rank -> same model
    sched = default_schedule(cfg, tp_size=tp)
    max_ctx = PROMPT_LEN + args.steps + args.warmup + 16
    plug = MegaKernelPlugin(cfg, sched, max_ctx=max_ctx, device=local, tp_rank=rank if tp > 1 else 0, tp_size=tp)
    plug.bind_weights(w)
    if tp > 1:
        from paper_2605_11581_b200.dist_utils import share_workspaces
        plug.bind_peers(share_workspaces(group, plug.workspace))
    cfg_bytes = full_cfg
    g = torch.Generator().manual_seed(1)
    prompt = torch.randint(0, full_cfg.vocab, (PROMPT_LEN,), generator=g).tolist()

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def prefill():
        # the decode path itself builds the prompt's KV cache (one launch per prompt token)
        prompt_dev = torch.tensor(prompt, dtype=torch.int32, device=dev)
        for p_, _ in enumerate(prompt[:-1]):
            plug.tokens.copy_(prompt_dev[p_:p_ + 1])
            plug.positions.fill_(p_)
            plug.enqueue(want_logits=False, auto_advance=False)
        plug.set_state(prompt[-1], PROMPT_LEN - 1)
        plug.check()

    # ---- device-resident loop: value + roofline ----
    prefill()
    for _ in range(args.warmup):
        plug.enqueue()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = plug.launches
    e0.record()
    for _ in range(args.steps):
        plug.enqueue()
    e1.record()
    barrier()
    plug.check()
    ms = e0.elapsed_time(e1) / args.steps
    launches = plug.launches - launches0

    # ---- end to end through the host-facing call ----
    prefill()
    tok, pos = prompt[-1], PROMPT_LEN - 1

    def e2e_step(tok, pos):
        # adamk_decode_step_host: H2D copy of (token, position) from pinned host memory, one launch, D2H copy of the
        # greedy token, stream synchronise -- one C-ABI call per token
        return plug.decode_step_host(tok, pos), pos + 1

    for _ in range(args.warmup):
        tok, pos = e2e_step(tok, pos)
    barrier()
    e0.record()
    for _ in range(args.steps):
        tok, pos = e2e_step(tok, pos)
    e1.record()
    barrier()
    plug.check()
    clocks = sampler.stop()
    ms_e2e = e0.elapsed_time(e1) / args.steps

    ms, ms_e2e = group.max_over_ranks([ms, ms_e2e], device=dev)
    if rank != 0:
        group.close()
        return

    peak, peak_kind = measured_peak()
    ctx_mid = PROMPT_LEN + args.warmup + args.steps // 2
    bytes_per_launch = cfg_bytes.algorithmic_bytes(ctx_mid) // tp   # per rank: one kernel streams 1/tp of the model
    achieved = bytes_per_launch / (ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():   # dram__bytes_read + write of one launch from an `ncu --set full` capture (not measurable inside this run)
        tj = json.loads(tfile.read_text())
        traffic, traffic_src = tj.get("dram_bytes_per_launch"), tj.get("source")
    line = base_line(args, full_cfg, world)
    jobs = 1 if tp > 1 else world               # tensor parallel: one sequence; replicas: one per GPU
    if tp > 1:
        line["scaling"] = "strong"
        line["config"]["parallelism"] = f"tp{tp} (in-kernel NVLink peer stores)"
    line.update({
        "value": jobs * 1e3 / ms, "ms_per_step": ms,
        "kernel": {"consumer_warps": sched.consumer_warps, "n_stage": sched.n_stage, "stage_bytes": sched.stage_bytes,
                   "inflight": sched.inflight, "fuse_down": sched.fuse_down, "n_sms": plug.n_sms},
        "e2e": {"value": jobs * 1e3 / ms_e2e, "unit": UNIT, "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 4,
                "ms_per_step": ms_e2e},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_kind": f"{peak_kind} copy bandwidth (burst)",
                     "algorithmic_bytes_per_launch": bytes_per_launch, "kernel": "adamk_decode_kernel",
                     "launch_ms": ms},
    })
    if tp == 1 and not args.no_prefill:
        line["prefill"] = prefill_sample(full_cfg, w, dev, local)
        line["batch_decode"] = batch_decode_sample(full_cfg, w, dev, local)
    if not args.no_cpu_baseline:
        w_cpu = random_weights(full_cfg, seed=0, device=dev).to("cpu") if tp > 1 else w.to("cpu")
        res = cpu_decode_sample(full_cfg, w_cpu, prompt, n_steps=args.cpu_steps)
        line["cpu_baseline"] = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line))
    group.close()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--cpu-steps", type=int, default=48, help="decode steps of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the extra tensor-core Prefill and batched-decode samples")
    ap.add_argument("--tp", action="store_true", help="N > 1: tensor-parallel shards of one sequence instead of N replicas")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        # `python bench.py --gpus N` outside torchrun: spawn the N ranks ourselves, one per GPU, NCCL rendezvous on
        # 127.0.0.1 (the driver's own launch line, reproduced)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
        raise SystemExit(subprocess.run(cmd).returncode)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
