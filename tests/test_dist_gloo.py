"""World-size-2 gloo test of the replica aggregation used by bench.py --gpus N."""

import os
import socket

import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2605_11581_b200.dist_utils import RankGroup

    g = RankGroup(backend="gloo")
    g.barrier()
    local_seconds = 0.5 + 0.25 * rank             # rank 1 is the slow replica
    mx = g.max_over_ranks([local_seconds, 10.0 - rank])
    agg = g.aggregate_throughput(units_per_rank=128, seconds_local=local_seconds)
    out.put((rank, mx, agg))
    g.close()


def test_replica_aggregation_world2():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(out.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, agg in results:
        assert mx == [0.75, 10.0]                  # max over ranks, element-wise
        assert abs(agg - 2 * 128 / 0.75) < 1e-9    # all ranks' tokens / slowest rank's time


def test_single_process_group_is_a_noop():
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        os.environ.pop(k, None)
    from paper_2605_11581_b200.dist_utils import RankGroup

    g = RankGroup()
    g.barrier()
    assert g.world == 1 and g.max_over_ranks([1.5]) == [1.5]
    assert g.aggregate_throughput(10, 2.0) == 5.0
