"""World-size-2 gloo tests of the multi-GPU plumbing (paper_1906_03420_b200/dist.py) on CPU.

The CUDA join cannot run here, so each rank's shard result comes from the oracle restricted
to that rank's contiguous, F-weighted slice of level-1 rows (root-restricted matching, the
same decomposition the device sharding uses); the collectives must then reproduce the
single-process result exactly and in order."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_1906_03420_b200 import dist as gd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        _body(rank, ws, out_q)
    except Exception as e:  # report instead of hanging the parent
        out_q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, ws, out_q):
    if True:
        res = {}
        # 1) graph replication through buffer views
        rng = np.random.default_rng(5)
        sizes = [1000, 0, 4096 * 3 + 7]
        if rank == 0:
            views = [torch.from_numpy(rng.integers(0, 255, s, dtype=np.uint8)) for s in sizes]
            meta = pickle.dumps({"sizes": sizes, "tag": "gsi"})
        else:
            views, meta = None, None

        def alloc_like(m):
            d = pickle.loads(m)
            return "graph", [torch.zeros(s, dtype=torch.uint8) for s in d["sizes"]]

        graph, views, meta = gd.broadcast_graph(meta, views, alloc_like)
        res["digest"] = [int(v.to(torch.int64).sum()) for v in views] + [len(meta)]
        # 2) sharded matching + count all-reduce + ordered table gather
        g = W.chung_lu(1500, 7000, 150, nlv=2, nle=2, seed=17)
        og = oracle.OracleGraph(g)
        qs = gd.broadcast_queries([W.random_walk_query(g, 4, 40 + i) for i in range(3)] if rank == 0 else None)
        counts = torch.zeros(len(qs), dtype=torch.int64)
        tables = []
        for i, q in enumerate(qs):
            roots = np.nonzero(g.vlabels == q.vlabels[0])[0]
            deg = np.bincount(np.concatenate([g.src, g.dst]), minlength=g.n)[roots]
            F = np.concatenate([[0], np.cumsum(deg)])          # work weight per level-1 row
            a, b = gd.shard_bounds(F, rank, ws)
            c, _, tab = oracle.match(og, q, root=0, roots=roots[a:b])
            counts[i] = c
            tables.append(gd.gather_tables(tab, q.n))
        gd.allreduce_counts(counts)
        res["counts"] = counts.tolist()
        res["tables"] = tables
        out_q.put((rank, res))


def test_gloo_world2_replication_shards_and_gather():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(ws))
    for r in range(ws):
        assert "error" not in got[r], got[r]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0]["digest"] == got[1]["digest"]
    g = W.chung_lu(1500, 7000, 150, nlv=2, nle=2, seed=17)
    og = oracle.OracleGraph(g)
    for i in range(3):
        qq = W.random_walk_query(g, 4, 40 + i)
        c, _, tab = oracle.match(og, qq, root=0)
        assert got[0]["counts"][i] == got[1]["counts"][i] == c
        assert np.array_equal(got[0]["tables"][i], tab)          # rank order == 1-process order
        assert got[1]["tables"][i] is None


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_partition(world):
    rng = np.random.default_rng(world)
    for trial in range(50):
        w = rng.integers(0, 50, rng.integers(1, 300))
        if trial % 7 == 0:
            w[rng.integers(len(w))] = 10_000                   # one hub row
        F = np.concatenate([[0], np.cumsum(w)])
        T = int(F[-1])
        bounds = [gd.shard_bounds(F, r, world) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == len(w)
        for r in range(world - 1):
            assert bounds[r][1] == bounds[r + 1][0]
        for r, (a, b) in enumerate(bounds):
            share = int(F[b] - F[a])
            assert share <= T / world + (w.max() if len(w) else 0) + 1
