"""ncu target: one tensor-core Prefill pass (default Qwen2.5-7B, 4096 tokens, 1 plane).  usage: prefill_launches.py [model] [T] [planes]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.plugin import MegaKernelPlugin
from paper_2605_11581_b200.prefill import TensorCorePrefill
from paper_2605_11581_b200.schedules import default_schedule
from paper_2605_11581_b200.weights import random_weights

cfg = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
planes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = random_weights(cfg, 0, device="cuda")
plug = MegaKernelPlugin(cfg, default_schedule(cfg), max_ctx=T + 16)
plug.bind_weights(w)
pre = TensorCorePrefill(cfg, w, plug, planes=planes, attention="bf16")
toks = torch.randint(0, cfg.vocab, (T,), device="cuda")
pre.run(toks)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prefill")
pre.run(toks)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
