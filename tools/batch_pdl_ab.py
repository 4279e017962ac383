"""A/B of the batched decode step with and without programmatic dependent launch (weights of each GEMM's first ring
pass issued ahead of griddepcontrol.wait), plus parity of the PDL path against the CPU oracle.
usage: batch_pdl_ab.py [quick]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2605_11581_b200.batch_decode as bd
from tools.batch_check import D128_Q3, TINY, bench, parity

if __name__ == "__main__":
    real = bd.BatchedDecoder

    import tools.batch_check as bc
    for mode in (0, 2, 3):
        class PdlDecoder(real):   # parity() builds its decoder with defaults: force the PDL mode for the check
            def __init__(self, *a, **kw):
                kw["pdl"] = mode
                super().__init__(*a, **kw)
        bc.BatchedDecoder = PdlDecoder
        print("pdl mode", mode, flush=True)
        parity(TINY, 3)
        parity(D128_Q3, 8)
        parity(D128_Q3, 8, oracle_cache=True)
    bc.BatchedDecoder = real
    if len(sys.argv) > 1 and sys.argv[1] == "quick":
        sys.exit(0)
    for rep in range(2):
        for B in (8, 16, 64):
            for pdl in (0, 2, 3):
                bench("qwen2.5-1.5b", B, 2048, pdl=pdl)
    bench("qwen2.5-1.5b", 8, 8192, pdl=0)
    bench("qwen2.5-1.5b", 8, 8192, pdl=3)
