"""Multi-GPU parity over NCCL: 2 ranks, one process per GPU.  Skipped when
fewer than 2 CUDA devices are visible (every GPU call of this run has one GPU; the host-side
logic is covered by the gloo tests in test_dist_cpu.py).

Rank 0 builds the graph and broadcasts its device buffers (gsi_graph_buffers -> NCCL broadcast
into gsi_graph_alloc_like on rank 1); both ranks run every query sharded (interleaved pieces);
the all-reduced counts and the gathered tables equal the 1-GPU results and the oracle.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if torch.cuda.device_count() < 2:
    pytest.skip("needs 2 CUDA devices", allow_module_level=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outq):
    import torch.distributed as dist

    import oracle
    import workloads as W
    from paper_1906_03420_b200 import dist as gd
    from paper_1906_03420_b200 import gsi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    g = W.chung_lu(20_000, 120_000, 2_000, nlv=8, nle=6, seed=91)
    qs = [W.random_walk_query(g, 4 + s % 5, 9100 + s) for s in range(8)]
    if rank == 0:
        graph = gsi.build(g, device=0)
        descs, meta = gsi.gsi_graph_buffers(graph)
        views = [gsi.torch_view(p, b, device="cuda:0") for (_, p, b) in descs]
    else:
        meta, views = None, None

    def alloc_like(m):
        gr, ds = gsi.gsi_graph_alloc_like(m, device=rank)
        return gr, [gsi.torch_view(p, b, device=f"cuda:{rank}") for (_, p, b) in ds]

    other, views, meta = gd.broadcast_graph(meta, views, alloc_like)
    if rank != 0:
        graph = other
    torch.cuda.synchronize()
    ok = True
    for q in qs:
        r = gsi.query(graph, q, want_table=True, shard_rank=rank, shard_count=world, shard_pieces=3)
        c = torch.tensor([r.count], dtype=torch.int64, device="cuda")
        gd.allreduce_counts(c)
        tab = gd.gather_tables(r.table(), q.n)
        if rank == 0:
            full = gsi.query(graph, q, want_table=True)
            cnt, fp, otab = oracle.match(oracle.OracleGraph(g), q)
            canon = lambda t: t[np.lexsort(t.T[::-1])] if len(t) else t
            ok &= int(c.item()) == full.count == cnt
            ok &= np.array_equal(canon(tab), otab)
    if rank == 0:
        outq.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_nccl_counts_and_tables():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
