"""N > 1 host-side path on CPU (gloo, world_size 2): one process per rank, each driving its own metadata-only pool
for its head shard (A19) through the C ABI with the same op script.  The allocator is replicated deterministically,
so ids, handles and tables agree across ranks with no data-path exchange — checked by an all_gather of table digests —
and bench.py's max/sum timing reduction is exercised with gloo."""
import hashlib
import os
import socket

import numpy as np
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


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2510_18586_b200 as tcb
        from workloads.configs import CONFIGS
        from workloads.replay import Replayer
        from workloads.scripts import build_script
        cfg = CONFIGS[name]
        pool = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, cfg.N, device=-1, shard_rank=rank, shard_world=world,
                        host_slots=cfg.host_slots(), max_blocks_per_agent=cfg.max_blocks_per_agent)
        assert pool.chunk_bytes == cfg.chunk_bytes(world)
        tr = Replayer(pool).run(build_script(cfg, 6))
        assert all(s == 0 for s, _ in tr)
        h = hashlib.sha256()
        for a in range(cfg.n_agents):
            h.update(np.asarray(pool.block_table(a), dtype=np.int32).tobytes())
        h.update(repr([x for _, x in tr]).encode())
        digest = torch.tensor(list(h.digest()), dtype=torch.uint8)
        got = [torch.empty_like(digest) for _ in range(world)]
        dist.all_gather(got, digest)
        same = all(torch.equal(g, got[0]) for g in got)
        # bench.py's reduction: max of per-rank times, sum of per-rank bytes
        my = torch.tensor([1.0 + rank, 100.0 * (rank + 1)], dtype=torch.float64)
        mx, sm = my.clone(), my.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        q.put((rank, same, float(mx[0]), float(sm[1]), pool.block_bytes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_head_sharded_ranks_agree_without_exchange(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[1] for r in res), "block tables diverged across ranks"
    assert all(r[2] == 2.0 and r[3] == 300.0 for r in res)
    from workloads.configs import CONFIGS
    assert res[0][4] == CONFIGS[name].block_bytes(world)
