"""Multi-rank host logic of the product-sharded path, on CPU:
world_size-2 torch.distributed over gloo (127.0.0.1).

Each rank builds a host-only plan (mf_options.host_only: the same C++ plan
logic the GPU ranks run, no device) for its shard, takes the products the plan
assigns it, forms its PARTIAL C = sum over its products of W[:,q] * P_q with the
oracle (P_q = T_q S_q from or_premix / or_classical), and the ranks sum the
partials with an all-reduce -- the exchange step that NCCL performs on GPUs.
The sum must be the exact product on integer inputs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mf_inputs
import oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, levels, n, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2312_12732_b200 as mf
        # bootstrap pattern of bench.py: rank 0's id bytes reach every rank
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        plan = mf.Plan(mf.triples.get(name), levels, n, shard_rank=rank, shard_count=world,
                       host_only=True)
        shard = plan.products()["shard"]
        mine = np.nonzero(shard == rank)[0]
        split = np.nonzero(shard == -1)[0]          # row-split leftovers
        r0, r1 = plan.shard_rows()
        # every rank sees the same assignment
        allsh = [None] * world
        dist.all_gather_object(allsh, shard.tolist())
        assert all(s == allsh[0] for s in allsh)

        F = oracle.kron_power(oracle.catalog(name), levels)
        A, B = mf_inputs.pair("int1024", n, 3)
        T, S = oracle.premix(A, F, "A"), oracle.premix(B, F, "B")
        P = np.zeros((F.R, n // F.p, n // F.p))
        for qq in mine:
            P[qq] = oracle.classical(T[qq], S[qq])
        Wm = F.W.copy()
        Wm[:, [qq for qq in range(F.R) if qq not in set(mine.tolist())]] = 0.0
        part = oracle.postmix(P, oracle.Triple("shard", F.p, F.U, F.V, Wm), n)
        if len(split):  # this rank's row slab [r0, r1) of every split product
            Ps = np.zeros_like(P)
            for qq in split:
                Ps[qq, r0:r1] = oracle.classical(T[qq], S[qq])[r0:r1]
            Ws = F.W.copy()
            Ws[:, [qq for qq in range(F.R) if qq not in set(split.tolist())]] = 0.0
            part = part + oracle.postmix(Ps, oracle.Triple("split", F.p, F.U, F.V, Ws), n)
        t = torch.from_numpy(part)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
        ok = bool((t.numpy() == exact).all())
        q.put((rank, ok, len(mine) + len(split) * (r1 - r0) / (n // F.p), shard.tolist()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(e), -1, None))


@pytest.mark.parametrize("name,levels,n", [("strassen-winograd", 2, 64), ("laderman", 1, 36),
                                           ("strassen-winograd", 1, 32),
                                           ("strassen-winograd", 2, 1024)])
def test_two_rank_partials_sum_to_product(name, levels, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, levels, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok, count, shard in res:
        assert ok is True, (rank, ok)
    counts = [r[2] for r in res]  # products per rank (split products count by row share)
    R = len(res[0][3])
    assert abs(sum(counts) - R) < 1e-9 and max(counts) - min(counts) <= 1  # balanced, complete
    assert set(res[0][3]) - {-1} == set(range(world))
