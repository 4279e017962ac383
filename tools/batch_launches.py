"""ncu target: one eager batched decode step.  usage: batch_launches.py [model] [B] [ctx]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200.batch_decode import BatchedDecoder
from paper_2605_11581_b200.model_config import PRESETS
from paper_2605_11581_b200.weights import random_weights

cfg = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-1.5b"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
w = random_weights(cfg, 0, device="cuda")
dec = BatchedDecoder(cfg, w, B, ctx + 64)
dec.set_state(torch.randint(0, cfg.vocab, (B,)).tolist(), [ctx] * B)
dec.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
dec.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
