"""World-size-2 gloo tests of the multi-GPU host path (CPU only).

The path has no data collective; what must hold across ranks is that the
shards tile the flat tensor exactly, that each rank's view addresses its own
range, and that the timing aggregation (sum of elements / max of times)
agrees on every rank."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_list, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_1909_07729_b200 import dist as kd
    r, lr, w = kd.init(backend="gloo")
    assert (r, w) == (rank, world)
    out = {}
    for n in n_list:
        b, c = kd.shard_range(n, w, r)
        # gather every rank's range; all ranks must see a gap-free tiling
        t = torch.tensor([b, c], dtype=torch.int64)
        parts = [torch.zeros(2, dtype=torch.int64) for _ in range(w)]
        dist.all_gather(parts, t)
        pos = 0
        for p in parts:
            assert int(p[0]) == pos or int(p[1]) == 0
            pos = int(p[0]) + int(p[1])
        assert pos == n
        # the view is this rank's slice of the flat tensor
        x = torch.arange(n, dtype=torch.int64)
        v = kd.shard_view(x, w, r)
        assert v.numel() == c and (c == 0 or (int(v[0]) == b and int(v[-1]) == b + c - 1))
        out[n] = (b, c)
    # aggregation: rank r "took" (r + 1) ms on (r + 1) * 1000 elements
    tot, ms, eps = kd.aggregate_throughput((r + 1) * 1000, float(r + 1))
    out["agg"] = (tot, ms, eps)
    out["gather"] = kd.gather_over_ranks([r, 10.0 * r + 0.5])
    kd.barrier()
    q.put((r, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shards_and_aggregation(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_list = [0, 1, 15, 16, 17, 65536, (1 << 24) + 3]
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_list, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for n in n_list:
        assert sum(res[r][n][1] for r in range(world)) == n
    # every rank computed the same whole-job numbers: 3000 elements / 2 ms
    for r in range(world):
        tot, ms, eps = res[r]["agg"]
        assert tot == 3000 and ms == 2.0 and abs(eps - 1.5e6) < 1e-6
        assert res[r]["gather"] == [[float(k), 10.0 * k + 0.5] for k in range(world)]
