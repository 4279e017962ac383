"""W4A16 (GPTQ-format int4) path: the byte model of the reference, the quantiser / reference dequantisation round trip,
the packed stream layout (CPU), and the MegaKernel against the oracle on the dequantised weights (GPU)."""

import json

import numpy as np
import pytest
import torch

from oracle.w4a16_ref import dequant_w4a16, dequantized_weights
from paper_2605_11581_b200 import quant, task_table as tt
from paper_2605_11581_b200.mkplan import graph_ir
from paper_2605_11581_b200.model_config import TINY, TINY_QWEN3, ModelConfig
from paper_2605_11581_b200.weights import random_weights

D128 = ModelConfig(name="test-d128", hidden=512, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=128, intermediate=1280, vocab=4096)
D128_Q3 = ModelConfig(name="test-d128-q3", hidden=512, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128, intermediate=1536,
                      vocab=3000, qkv_bias=False, qk_norm=True, tied_embed=False)
SCHED = tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2, attn_min_chunk=16, l2_prefetch_kb=64,
                          inflight=2, fuse_down=True, w4a16=True)
SCHED8 = tt.KernelSchedule(consumer_warps=8, n_stage=4, rows_per_tile=16, ktile_chunks=2, attn_min_chunk=8, fuse_down=True, w4a16=True)


def test_quantiser_round_trip_and_byte_model():
    """dequant(quantize(W)) is within half a step of W, re-quantising is the identity, and the container holds exactly
    the bytes the reference's model charges (graph_ir.py:296-305: n * k / 2 codes + n * ceil(k / 128) * 2 scale bytes)."""
    g = torch.Generator().manual_seed(0)
    for n, k in ((64, 256), (10, 1536), (33, 200), (5, 8)):
        w = (torch.randn(n, k, generator=g) * 0.05).to(torch.bfloat16)
        m = quant.quantize_matrix(w)
        d = dequant_w4a16(m.q, m.s)
        step = m.s.float().repeat_interleave(128, dim=1)[:, :k]
        assert ((d - w.float()).abs() <= 0.5 * step + 1e-6).all()
        m2 = quant.quantize_matrix(d.to(torch.float32))
        assert torch.equal(dequant_w4a16(m2.q, m2.s), d)
        graph = {"buffers": [{"id": "x", "space": "SharedPage", "bytes": 16 * k * 2}, {"id": "w", "space": "Global", "bytes": n * k * 2},
                             {"id": "y", "space": "Global", "bytes": 16 * n * 2}],
                 "operators": [{"id": "g", "kind": "Gemm", "dims": {"m": 1, "n": n, "k": k}, "dtype": "int4_w4a16", "inputs": ["x"],
                                "outputs": ["y"], "weight": "w"}]}
        op = graph_ir.load_graph(json.dumps(graph)).operators[0]
        assert m.nbytes() == graph_ir.weight_bytes(op) == n * k // 2 + n * -(-k // 128) * 2
        assert graph_ir.scale_bytes(op) == m.s.numel() * 2


@pytest.mark.parametrize("cfg,sched", [(TINY, SCHED), (D128_Q3, SCHED8)], ids=["tiny", "d128-q3"])
def test_int4_stream_covers_every_code_and_scale(cfg, sched):
    """Invert the packed int4 stream: every code of every projection matrix appears exactly once, next to its scale."""
    table = tt.build_task_table(cfg, sched)
    qw = quant.quantize_weights(random_weights(cfg, seed=3))
    packed = tt.pack_weights_reference(table, qw).view(np.uint8)
    assert packed.nbytes == table.packed_weight_bytes
    seen = {}
    for task in table.tasks:
        ttype, aux = int(task[tt.F_TYPE]), int(task[tt.F_AUX])
        if ttype == tt.T_LMHEAD:
            assert not aux & tt.AUX_INT4
            continue
        if ttype not in tt.STREAM_TYPES:
            continue
        assert aux & tt.AUX_INT4
        layer, pos = int(task[tt.F_LAYER]), int(task[tt.F_WOFF]) * 16
        if ttype == tt.T_DOWNK:
            k0, nk, h = int(task[tt.F_A]), int(task[tt.F_B]), int(task[tt.F_K])
            qm = qw.layers[layer]["wdown"]
            g0, ng = k0 // 128, tt.downk_i4_groups(k0, nk)
            sc = packed[pos:pos + ng * h * 2].view(np.uint16).reshape(ng, h)
            assert (sc == qm.s.numpy().view(np.uint16)[:, g0:g0 + ng].T).all()
            pos += ng * h * 2
            codes = dequant_codes(qm)
            for j in range(nk):
                col = packed[pos:pos + h // 2]
                got = np.empty(h, dtype=np.uint8)
                got[0::2], got[1::2] = col & 15, col >> 4
                assert (got == codes[:, k0 + j]).all()
                cover = seen.setdefault((layer, "wdown"), np.zeros(codes.shape, dtype=np.int32))
                cover[:, k0 + j] += 1
                pos += h // 2
            continue
        vrow0, k, rt, ktc = int(task[tt.F_A]), int(task[tt.F_K]), int(task[tt.F_RT]), int(task[tt.F_KTC])
        lane = np.arange(32)
        for tile, kt, rows, chunks in tt.stage_shapes(task):
            for r in range(rows):
                name, row = tt.virtual_row_source(cfg, ttype, vrow0 + tile * rt + r)
                qm = qw.layers[layer][name]
                codes = dequant_codes(qm)
                cover = seen.setdefault((layer, name), np.zeros(codes.shape, dtype=np.int32))
                for c in range(chunks):
                    blk, kbase = r * chunks + c, (kt * ktc + c) * tt.KCHUNK
                    words = packed[pos + blk * 128:pos + (blk + 1) * 128].view("<u4")
                    for el in range(8):
                        kidx = kbase + (4 * lane + el if el < 4 else 128 + 4 * lane + el - 4)
                        got = (words >> (4 * el)) & 15
                        ok = kidx < k
                        assert (got[ok] == codes[row, kidx[ok]]).all() and (got[~ok] == 8).all()
                        cover[row, kidx[ok]] += 1
                    sc = packed[pos + rows * chunks * 128 + blk * 4:pos + rows * chunks * 128 + blk * 4 + 4].view(np.uint16)
                    srow = qm.s[row].numpy().view(np.uint16)
                    for gi in range(2):
                        g = kbase // 128 + gi
                        assert sc[gi] == (srow[g] if g < srow.size else 0)
            pos += tt.i4_stage_bytes(rows, chunks)
    assert len(seen) == 7 * cfg.n_layers
    for key, cover in seen.items():
        assert (cover == 1).all(), key


def dequant_codes(qm) -> np.ndarray:
    q = qm.q.numpy()
    out = np.empty((q.shape[0], q.shape[1] * 2), dtype=np.uint8)
    out[:, 0::2], out[:, 1::2] = q & 15, q >> 4
    return out


def test_w4a16_schedule_validation_and_bytes():
    with pytest.raises(tt.ScheduleError):
        tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2, w4a16=True)       # needs fuse_down
    from paper_2605_11581_b200.model_config import QWEN25_1P5B as cfg
    sched = tt.KernelSchedule(consumer_warps=7, n_stage=5, rows_per_tile=42, ktile_chunks=2, attn_min_chunk=112, inflight=3, fuse_down=True, w4a16=True)
    table = tt.build_task_table(cfg, sched)
    layer_elems = cfg.n_layers * (cfg.qkv_rows * cfg.hidden + cfg.hidden * cfg.q_dim + 3 * cfg.intermediate * cfg.hidden)
    lm = cfg.vocab * cfg.hidden * 2
    # codes are half a byte per element; scales, K padding and 16-byte stage alignment add a few per cent
    assert layer_elems // 2 + lm <= table.packed_weight_bytes <= int(layer_elems * 0.55) + lm


# ---------------------------------------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("cfg,sched", [(TINY, SCHED), (TINY_QWEN3, SCHED8), (D128, SCHED), (D128_Q3, SCHED), (D128_Q3, SCHED8)],
                         ids=["tiny-c7", "tiny-q3-c8", "d128-c7", "d128-q3-c7", "d128-q3-c8"])
def test_w4a16_decode_matches_oracle_on_dequantised_weights(cfg, sched):
    """Teacher-forced decode with int4 weights: logits of the MegaKernel (codes and scales streamed through the ring,
    dequantised in the consumer warps) against the CPU oracle run on the fp32 dequantisation of the same codes."""
    from oracle.decode_ref import RefDecoder
    from paper_2605_11581_b200.plugin import MegaKernelPlugin
    from paper_2605_11581_b200.weights import rope_table

    max_ctx = 128
    qw = quant.quantize_weights(random_weights(cfg, seed=0))
    cos, sin = rope_table(cfg, max_ctx)
    ref = RefDecoder(cfg, dequantized_weights(qw), max_ctx, cos, sin)
    plug = MegaKernelPlugin(cfg, sched, max_ctx=max_ctx)
    plug.bind_weights(qw)
    want_packed = tt.pack_weights_reference(plug.table, qw).view(np.uint8)
    got_packed = plug.packed[:plug.table.packed_weight_bytes].cpu().numpy()
    assert (got_packed == want_packed).all()                       # the device packer is bit-exact
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, cfg.vocab, (40,), generator=g).tolist()
    worst = 0.0
    for pos, tok in enumerate(toks):
        want = ref.step([tok], [pos])[0].numpy()
        out = plug.decode_step(tok, pos, want_logits=True)
        plug.check()
        got = out.logits[0].cpu().numpy()
        err = float(np.abs(got - want).max())
        worst = max(worst, err)
        assert err <= 2e-3, (pos, err)
        srt = np.sort(want)
        if srt[-1] - srt[-2] > 1e-2:
            assert int(out.next_token.item()) == int(want.argmax()), pos
    print(f"w4a16 {cfg.name}: max |logit diff| vs oracle {worst:.2e}")
    plug.close()
