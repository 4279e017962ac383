"""Where a decode-sized GEMM launch spends its time: %globaltimer stamps of CTA 0 (adamk_prefill_set_trace)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2605_11581_b200 import prefill as P

lib = P._lib()
B, H, I = 8, 1536, 8960
x = torch.randn(2, B, H, device="cuda").to(torch.bfloat16)
a = torch.randn(2, B, I, device="cuda").to(torch.bfloat16)
shapes = {"qkv 1536->2048": (x, (torch.randn(2048, H, device="cuda") / H ** 0.5).to(torch.bfloat16)),
          "gate/up 1536->17920": (x, (torch.randn(2 * I, H, device="cuda") / H ** 0.5).to(torch.bfloat16)),
          "down 8960->1536": (a, (torch.randn(H, I, device="cuda") / I ** 0.5).to(torch.bfloat16))}
stamps = torch.zeros(16, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["prologue", "first operands", "k loop", "epilogue", "teardown wait"]
tile = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for name, (xp, w) in shapes.items():
    out = torch.zeros(B, w.shape[0], device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    acc, tot, seen = [0.0] * 5, 0.0, 0.0
    n = 20
    for it in range(n + 3):
        flush.zero_()                       # weights out of L2, as in a real step
        lib.adamk_prefill_set_trace(P._ptr(stamps))
        e0.record()
        P.gemm(xp, w, out, epilogue=P.EPI_ATOMIC, tile_n=tile)
        e1.record()
        lib.adamk_prefill_set_trace(None)
        torch.cuda.synchronize()
        if it >= 3:
            t = stamps.tolist()
            for i in range(5):
                acc[i] += (t[i + 1] - t[i]) / 1e3
            seen += (t[6] - t[3]) / 1e3          # commit issued -> accumulator visible to the epilogue warp
            tot += e0.elapsed_time(e1) * 1e3
    print(f"tile {tile} {name}: event {tot / n:.1f} us | CTA 0: " + ", ".join(f"{names[i]} {acc[i] / n:.2f}" for i in range(5)) +
          f" | sum {sum(acc) / n:.2f} us | of the epilogue, waiting for the MMAs to retire: {seen / n:.2f}", flush=True)
