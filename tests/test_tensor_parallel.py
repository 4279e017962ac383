"""Tensor-parallel sharding: host logic on the CPU -- the shards, the sharded oracle against
the unsharded one, and a world-size-2 gloo run in which each process owns one rank and the partial sums are
all-reduced.  The GPU side (in-kernel peer stores) is tested in tests/test_gpu_decode.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2605_11581_b200 import task_table as tt
from paper_2605_11581_b200.model_config import QWEN25_1P5B, QWEN3_8B, ModelConfig
from paper_2605_11581_b200.weights import random_weights, rope_table

CFG = ModelConfig(name="test-tp", hidden=256, n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=64,
                  intermediate=512, vocab=1024, qkv_bias=True, qk_norm=True, tied_embed=False)


def test_shard_dimensions_and_errors():
    lc = QWEN3_8B.shard(8)
    assert (lc.n_q_heads, lc.n_kv_heads, lc.intermediate, lc.vocab, lc.hidden) == (4, 1, 1536, 18992, 4096)
    assert QWEN25_1P5B.shard(2).n_kv_heads == 1
    with pytest.raises(ValueError):
        QWEN25_1P5B.shard(4)          # 2 kv heads do not split 4 ways: "replicas only" beyond TP = 2
    with pytest.raises(ValueError):
        QWEN3_8B.shard(3)
    # every rank's task table covers its shard; the byte streams of the ranks add up to the whole model
    tables = [tt.build_task_table(lc, tt.KernelSchedule(consumer_warps=7, n_stage=3, rows_per_tile=56, ktile_chunks=2))
              for _ in range(1)]
    full = QWEN3_8B
    per_rank = tables[0].packed_weight_bytes
    whole = 2 * (full.n_layers * (full.qkv_rows * full.hidden + full.hidden * full.q_dim + 3 * full.intermediate * full.hidden)
                 + full.vocab * full.hidden)
    assert per_rank * 8 == whole


def test_weight_shards_tile_the_matrices():
    w = random_weights(CFG, seed=4)
    for tp in (2, 4):
        shards = [w.shard(r, tp) for r in range(tp)]
        for l in range(CFG.n_layers):
            assert torch.equal(torch.cat([s.layers[l].wq for s in shards]), w.layers[l].wq)
            assert torch.equal(torch.cat([s.layers[l].wk for s in shards]), w.layers[l].wk)
            assert torch.equal(torch.cat([s.layers[l].bv for s in shards]), w.layers[l].bv)
            assert torch.equal(torch.cat([s.layers[l].wo for s in shards], dim=1), w.layers[l].wo)
            assert torch.equal(torch.cat([s.layers[l].wup for s in shards]), w.layers[l].wup)
            assert torch.equal(torch.cat([s.layers[l].wdown for s in shards], dim=1), w.layers[l].wdown)
        assert torch.equal(torch.cat([s.lm_head for s in shards]), w.lm_head_matrix)
        assert all(s.embed is w.embed for s in shards)


@pytest.mark.parametrize("tp", [2, 4])
def test_sharded_oracle_matches_unsharded(tp):
    from oracle.decode_ref import RefDecoder
    from oracle.tp_ref import RankRef, tp_step

    w = random_weights(CFG, seed=0)
    cos, sin = rope_table(CFG, 64)
    ref = RefDecoder(CFG, w, 64, cos, sin)
    ranks = [RankRef(CFG, w, r, tp, 64, cos, sin) for r in range(tp)]
    g = torch.Generator().manual_seed(3)
    for pos, tok in enumerate(torch.randint(0, CFG.vocab, (12,), generator=g).tolist()):
        want = ref.step([tok], [pos])[0]
        got = tp_step(ranks, tok, pos)
        assert torch.allclose(got, want, atol=2e-4, rtol=1e-4), (pos, float((got - want).abs().max()))
        assert int(got.argmax()) == int(want.argmax())


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle.tp_ref import RankRef, tp_step
    from paper_2605_11581_b200.dist_utils import RankGroup

    torch.set_num_threads(1)
    grp = RankGroup(backend="gloo")
    w = random_weights(CFG, seed=0)
    cos, sin = rope_table(CFG, 64)
    me = RankRef(CFG, w, rank, world, 64, cos, sin)

    def reduce(part):
        t = part.clone()
        dist.all_reduce(t)
        return t

    toks, outs = [5, 77, 1000, 3, 512, 9], []
    for pos, tok in enumerate(toks):
        local = tp_step([me], tok, pos, reduce=reduce)            # this rank's vocabulary slice
        best = torch.tensor([float(local.max()), float(local.argmax() + rank * me.cfg.vocab)], dtype=torch.float64)
        gathered = [torch.zeros_like(best) for _ in range(world)]
        dist.all_gather(gathered, best)                            # the (value, index) exchange of the kernel
        outs.append(int(max(gathered, key=lambda t: (float(t[0]), -float(t[1])))[1]))
    out.put((rank, outs))
    grp.close()


def test_two_process_tensor_parallel_over_gloo():
    """world_size 2 on the CPU: each process owns one rank, partial sums go through all_reduce, the argmax
    through an all_gather of (value, index) pairs; both ranks end with the unsharded oracle's tokens."""
    from oracle.decode_ref import RefDecoder

    w = random_weights(CFG, seed=0)
    cos, sin = rope_table(CFG, 64)
    ref = RefDecoder(CFG, w, 64, cos, sin)
    want = [int(ref.step([tok], [pos])[0].argmax()) for pos, tok in enumerate([5, 77, 1000, 3, 512, 9])]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == want and results[1] == want
