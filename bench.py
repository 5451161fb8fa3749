#!/usr/bin/env python
"""bench.py — GSI subgraph matching on B200: matches/s and ms/query (BASELINE.json metric).

One "step" = one pass of the whole hot path (filter -> plan -> every join level, SURVEY.md
§8(a)) over one batch of Q seeded random-walk queries against a
seeded synthetic data graph shaped like the paper's workloads.  The graph
(PCSR + signatures, tens of GB) is built once, outside the timed region, like the paper's
offline preprocessing; it is far larger than the 126 MB L2, so no L2
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5b] [--queries Q]
  python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)

Multi-GPU (torchrun, one rank per GPU): rank 0 builds the graph and broadcasts its device
buffers over NCCL; every query's rows are sharded across ranks and the
per-query counts are all-reduced (NCCL) — total work is fixed, so scaling is "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

# Workloads.  C5b is the join-stress scale-free config the HBM target is
# evaluated on; the others are selectable for context.
BENCH_CONFIGS = {
    "C2": dict(kind="C2", desc="enron-shaped Chung-Lu n=36692 m=183831 |L_V|=10 |L_E|=100"),
    "C3": dict(kind="C3", desc="gowalla-shaped Chung-Lu n=196591 m=950327 |L_V|=|L_E|=100"),
    "C4": dict(kind="C4", desc="road-shaped lattice 3742^2 m=17M |L_V|=|L_E|=1000"),
    "C5a": dict(kind="C5a", desc="R-MAT scale 25 ef 8 (~250M E) |L_V|=1000 |L_E|=86"),
    "C5b": dict(kind="C5b", desc="R-MAT scale 25 ef 8 (~250M E) |L_V|=10 |L_E|=86"),
    "C5m": dict(kind="C5m", desc="R-MAT scale 25 ef 8 (~264M E) |L_V|=100 |L_E|=86 (join-stress, bounded)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nme, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nme)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_workload(cfg: str, nq: int, k: int, device: str, seed: int = 1, scale: int | None = None):
    t0 = time.time()
    kind = BENCH_CONFIGS[cfg]["kind"]
    over = {}
    if scale is not None and kind.startswith("C5"):
        over["scale"] = scale
    g = W.make_config(kind, seed=seed, device=device, **over)
    t1 = time.time()
    adj = W._Adj(g, device=device)
    qs = [W.random_walk_query(g, k, 1000 + i, adj) for i in range(nq)]
    del adj
    log(f"[bench] workload {cfg}: n={g.n} m={g.m} gen {t1 - t0:.1f}s queries {time.time() - t1:.1f}s")
    return g, qs


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------ CPU oracle -----
def oracle_sample(og, qs, budget_s: float, per_query_timeout: float, threads: int, start: int = 0):
    """Run the oracle (as it stands) over queries start, start+1, ... until budget_s elapses.
    Returns (matches, seconds, queries_done, timeouts)."""
    import oracle
    matches, secs, done, touts = 0, 0.0, 0, 0
    i = start
    while secs < budget_s and done < len(qs):
        q = qs[i % len(qs)]
        t = time.perf_counter()
        c, fp, _ = oracle.match(og, q, table=False, threads=threads, timeout=per_query_timeout, partial=True)
        el = time.perf_counter() - t
        if per_query_timeout > 0 and el >= per_query_timeout:
            touts += 1
        secs += el
        matches += c
        done += 1
        i += 1
    return matches, secs, done, touts


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    import oracle
    dev = "cuda" if _cuda_ok() else "cpu"
    g, qs = make_workload(args.config, args.queries, args.k, dev, scale=args.scale)
    t = time.time()
    og = oracle.OracleGraph(g)
    log(f"[bench] oracle index {time.time() - t:.1f}s")
    threads = len(os.sched_getaffinity(0))
    per_step = args.ref_step_budget
    for _ in range(args.warmup):
        oracle_sample(og, qs, min(per_step, 2.0), args.ref_query_timeout, threads)
    tot_m, tot_s, tot_q, tot_to = 0, 0.0, 0, 0
    pos = 0
    for _ in range(args.steps):
        m, s, d, to = oracle_sample(og, qs, per_step, args.ref_query_timeout, threads, start=pos)
        pos += d
        tot_m += m; tot_s += s; tot_q += d; tot_to += to
    value = tot_m / tot_s if tot_s > 0 else 0.0
    line = {
        "impl": "reference", "metric": "matches/s", "value": value, "unit": "matches/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot_s / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": workload_config(args, g),
        "ms_per_query": 1000.0 * tot_s / max(tot_q, 1),
        "cpu_baseline": {"value": value, "unit": "matches/s", "cores": threads, "kind": "oracle",
                         "sample": f"{tot_q} queries of the batch (cycled), per-query timeout "
                                   f"{args.ref_query_timeout}s ({tot_to} timed out, partial counts kept), "
                                   f"~{per_step}s per step"},
        "e2e": {"value": value, "unit": "matches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def workload_config(args, g):
    return {"workload": f"{args.config}: {BENCH_CONFIGS[args.config]['desc']}", "n": int(g.n), "m": int(g.m),
            "queries_per_step": args.queries, "query_k": args.k, "query_seeds": f"1000..{999 + args.queries}",
            "graph_seed": 1,
            "mode": {"fp": "fingerprint (every match of the last level produced on the device, its candidate "
                           "read and checked, the match hashed into the order-free set fingerprint; no "
                           "closed-form counting)",
                     "count": "count (closed-form last two levels, DESIGN.md §6 count-ahead)",
                     "table": "table (every match written to HBM, query-id order)"}[args.mode],
            "l2": "inputs larger than L2 (PCSR+signatures >> 126 MB); no flush",
            "concurrency": args.concurrency}


# ------------------------------------------------------------------------ GPU arm --------
def run_gsi(args):
    import torch
    import torch.distributed as dist
    from paper_1906_03420_b200 import gsi

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # ---- small queries (C2 enron-shaped, C4 road-shaped): per-query latency, measured first
    # in a clean process (no 20 GB graph or grown workspace of the big workload resident) ----
    small = None
    if ws == 1 and not args.no_small:
        small = {}
        for cfg in args.small_configs:
            small[cfg] = small_query_latency(gsi, cfg, args.queries, args.k, local)
    # ---- the oracle single-threaded on C1-C3 (a baseline, not the target) --
    cpu_single = None
    if ws == 1 and not args.no_small and rank == 0:
        cpu_single = oracle_single_thread(args.queries, args.k)

    # ---- workload + graph (rank 0 builds; replicas via NCCL broadcast) ----------------
    if rank == 0:
        g, qs = make_workload(args.config, args.queries, args.k, "cuda", scale=args.scale)
        t = time.time()
        graph = gsi.build(g, device=local)
        torch.cuda.synchronize()
        info = graph.info()
        log(f"[bench] gsi_build_graph {time.time() - t:.2f}s: groups={info['n_groups']} "
            f"max_chain={info['max_chain']} bytes={info['bytes_total'] / 1e9:.2f} GB")
    if ws > 1:
        from paper_1906_03420_b200 import dist as gd
        t = time.time()
        if rank == 0:
            descs, meta = gsi.gsi_graph_buffers(graph)
            views = [gsi.torch_view(p, b, device=f"cuda:{local}") for (_, p, b) in descs]
        else:
            meta, views = None, None

        def alloc_like(m):
            gr, ds = gsi.gsi_graph_alloc_like(m, device=local)
            return gr, [gsi.torch_view(p, b, device=f"cuda:{local}") for (_, p, b) in ds]

        other, views, meta = gd.broadcast_graph(meta, views, alloc_like)
        if rank != 0:
            graph = other
        qarr = gd.broadcast_queries([(q.vlabels, q.src, q.dst, q.elabels) for q in qs] + [(g.n, g.m)]
                                    if rank == 0 else None)
        if rank != 0:
            nm = qarr[-1]
            qs = [W.Query(len(a[0]), *a) for a in qarr[:-1]]
            g = W.Graph(nm[0], np.zeros(0), np.zeros(nm[1]), np.zeros(nm[1]), np.zeros(nm[1]))
        torch.cuda.synchronize()
        if rank == 0:
            log(f"[bench] NCCL broadcast of the graph {time.time() - t:.2f}s")
    info = graph.info()

    shard = dict(shard_rank=rank, shard_count=ws, shard_pieces=args.shard_pieces) if ws > 1 else {}
    prepared = [gsi.prepare(graph, q) for q in qs]
    counts = torch.zeros(len(qs), dtype=torch.int64, device="cuda")
    MODES = {"count": dict(fingerprint=False),                    # the count path (closed-form last level)
             "fp": dict(fingerprint=True),                        # every final match read and hashed
             "table": dict(fingerprint=False, want_table=True)}   # every final match written (query-id order)

    def step(mode="count", profile=False, stats=None, which=None, timeout=None, sh=None, conc=None):
        """One pass of the hot path over the batch (or the queries `which`).  The batch runs its
        queries concurrently (--concurrency host workers / streams); the profiled pass runs them
        one at a time so per-kernel event times are not shared."""
        ps = prepared if which is None else [prepared[i] for i in which]
        rs = gsi.gsi_query_run_batch(graph, ps, concurrency=1 if profile else (conc or args.concurrency),
                                     timeout_s=args.query_timeout if timeout is None else timeout, profile=profile,
                                     partial_on_timeout=True, **MODES[mode], **(shard if sh is None else sh))
        c = torch.tensor([r.count for r in rs], dtype=torch.int64, device="cuda")
        if stats is not None:
            stats.extend(r.stats() for r in rs)
        if which is None:
            counts.copy_(c)
            c = counts
        if ws > 1 and sh is None:
            dist.all_reduce(c)
        return c

    def e2e_step():
        # the public API from host arrays: validate + encode + H2D of every query, the
        # concurrent batch run, and the counts back on the host
        ps = [gsi.prepare(graph, q) for q in qs]
        rs = gsi.gsi_query_run_batch(graph, ps, concurrency=args.concurrency, timeout_s=args.enum_timeout,
                                     partial_on_timeout=True, **MODES[args.mode], **shard)
        counts.copy_(torch.tensor([r.count for r in rs], dtype=torch.int64))
        if ws > 1:
            dist.all_reduce(counts)
        return int(counts.sum().item())

    def timed(fn):
        """Device time of fn() on the launching stream, max over ranks (ms)."""
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    HEAD = args.mode   # the headline pass: "fp" = every match produced, read and hashed
    for _ in range(args.warmup):
        step(HEAD, timeout=args.enum_timeout)
    torch.cuda.synchronize()
    per_query_counts = step(HEAD, timeout=args.enum_timeout).tolist()
    total_matches = int(sum(per_query_counts))

    # ---- timed region: device-timed, prepared (resident) queries ------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launch_stats = []
    with ClockSampler(local) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step(HEAD, stats=launch_stats, timeout=args.enum_timeout)
        ev1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    value = total_matches * args.steps / (ms / 1000.0)
    launches = sum(s["total_launches"] for s in launch_stats)
    capped = sum(s["capped"] for s in launch_stats) / args.steps
    q_ms = np.array([s["ms_total"] for s in launch_stats])
    q_ms_by_query = q_ms.reshape(args.steps, len(qs)).mean(axis=0)

    # ---- e2e: public API from host arrays, H2D of the query + D2H of the count -----------
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        m_e2e = e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    h2d = sum(4 * q.n + 12 * len(q.src) + 64 * q.n for q in qs)        # query arrays + signatures
    d2h = sum(8 * q.n + 64 * (2 * q.n + 2) for q in qs)                # |C(u)|, per-level sizes, count

    # ---- count-only: the library's default count path (the last two levels in closed form
    # per row of M_{k-2}, DESIGN.md §6 count-ahead) -- per-query latency, not join throughput
    count_only = None
    if not args.no_count_only:
        c_stats = []
        c_ms, c_counts = timed(lambda: step("count", stats=c_stats))
        c_counts = c_counts.tolist()
        c_q = np.array([s_["ms_total"] for s_ in c_stats])
        count_only = {"value": sum(c_counts) / (c_ms / 1000.0), "unit": "matches/s", "ms_per_step": c_ms,
                      "ms_per_query": c_ms / len(qs), "query_ms_p50": float(np.percentile(c_q, 50)),
                      "query_ms_p95": float(np.percentile(c_q, 95)),
                      "capped_queries": int(sum(s_["capped"] for s_ in c_stats)),
                      "counts_equal_headline": c_counts == per_query_counts,
                      "note": "count-only gsi_query (C ABI default): the last two levels are counted in closed "
                              "form per row of M_{k-2} (|L|-[inj in L] survivors x (|RR| - row hits) extensions), "
                              "so no per-match work; reported for ms/query, not as join throughput"}

    # ---- table: every match written to HBM as a k-int32 row in query-id order -------------
    table = None
    if not args.no_table:
        row_b = 4 * args.k
        which = [i for i, c in enumerate(per_query_counts) if 0 < c * row_b <= args.table_max_gb * 1e9]
        if which:
            t_stats = []
            gsi.gsi_trim_workspace(local)   # the tables need the memory the count passes reserved
            step("table", which=which, timeout=args.enum_timeout, conc=1)   # warm-up (workspace regrowth)
            t_ms, t_counts = timed(lambda: step("table", stats=t_stats, which=which, timeout=args.enum_timeout,
                                                conc=1))
            t_m = int(t_counts.sum().item())
            table = {"value": t_m / (t_ms / 1000.0), "unit": "matches/s", "ms": t_ms, "queries": which,
                     "matches": t_m, "GB_written": t_m * row_b / 1e9,
                     "write_GBps": t_m * row_b / 1e9 / (t_ms / 1000.0),
                     "counts_equal_headline": t_counts.tolist() == [per_query_counts[i] for i in which],
                     "kernel_variants": _variants(t_stats),
                     "note": f"want_table on the bench queries whose table fits {args.table_max_gb} GB "
                             f"(4k B per match, device-resident)"}

    # ---- profiled pass: per-kernel-variant CUDA-event times + algorithmic bytes ------------
    pstats = []
    step(HEAD, profile=True, stats=pstats, timeout=args.enum_timeout)
    torch.cuda.synchronize()
    ms_k, bytes_k, launches_k = np.zeros(8), np.zeros(8), np.zeros(8)
    nv = gsi.GSI_N_KVARIANT
    ms_v, bytes_v, launches_v = np.zeros(nv), np.zeros(nv), np.zeros(nv)
    for s in pstats:
        ms_k += np.array(s["ms_kernel"])
        bytes_k += np.array(s["alg_bytes"])
        launches_k += np.array(s["launches"])
        ms_v += np.array(s["ms_variant"])
        bytes_v += np.array(s["alg_bytes_variant"])
        launches_v += np.array(s["variant_launches"])
    items_v = np.zeros(nv)
    for s in pstats:
        items_v += np.array(s["items_variant"], dtype=np.float64)
    dom = int(np.argmax(ms_v))
    dname = gsi.KVARIANT[dom]
    peak, peak_src = load_peaks()
    clk_mhz = clk.summary().get("sm_mhz") or 1965.0
    # ncu evidence of this workload (profiles/ncu_traffic.json, tools/ncu_traffic.py): DRAM bytes
    # per launch, and the ALU-pipe activity of the k_final_fp capture
    tt_all = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tt_all = json.load(open(tp)).get(args.config, {})

    def hbm_entry(i):
        nm = gsi.KVARIANT[i]
        ach = (bytes_v[i] / (ms_v[i] / 1e3)) / 1e9 if ms_v[i] > 0 else 0.0
        tt = tt_all.get(nm, {})
        return {"bound": "hbm", "kernel": nm, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": tt.get("dram_bytes_per_launch"), "traffic_source": tt.get("source"),
                "ncu_dram_frac": tt.get("dram_frac"),
                "alg_bytes_per_launch": float(bytes_v[i] / max(launches_v[i], 1)),
                "ms_per_launch": float(ms_v[i] / max(launches_v[i], 1)), "peak_source": peak_src,
                "share_of_step": float(ms_v[i] / max(ms_k.sum(), 1e-9))}

    if dname == "final_fp":
        # integer-ALU bound: per match the fingerprint spec needs two splitmix
        # finalisers (their leading constant add folded into the row's partial sum) and four
        # 64-bit add/xor combines; on the 32-bit ALU pipe (SHF / LOP3 / IADD3; the multiplies run
        # on the FMA pipe) that is 2 x 3 xorshifts x 4 + 4 x 2 = FP_ALU_OPS lane-ops per match
        # (ncu's ALU-pipe activity of the kernel is reported beside the fraction).
        # Peak = 148 SMs x 4 SMSPs x 16 lanes/clk (ALU pipe, rt = 2) x the SM clock under load.
        FP_ALU_OPS = 32
        ops = items_v[dom] * FP_ALU_OPS
        ach = ops / (ms_v[dom] / 1e3) / 1e9
        pk = 148 * 4 * 16 * clk_mhz * 1e6 / 1e9
        tt = tt_all.get(dname, {})
        roofline = {"bound": "alu", "kernel": dname, "achieved": ach, "peak": pk, "unit": "Gop/s",
                    "frac": ach / pk, "traffic": tt.get("dram_bytes_per_launch"),
                    "traffic_source": tt.get("source"), "ncu_alu_pipe_active": tt.get("alu_pipe_active"),
                    "ncu_issue_active": tt.get("issue_active"),
                    "matches_per_launch": float(items_v[dom] / max(launches_v[dom], 1)),
                    "ms_per_launch": float(ms_v[dom] / max(launches_v[dom], 1)),
                    "peak_source": f"derived: 148 SMs x 4 SMSPs x 16 ALU lanes/clk x {clk_mhz:.0f} MHz "
                                   "(B300_MICROARCH.md pipe rates; B200_PROFILING.md SM count/clock)",
                    "ops_per_match": FP_ALU_OPS,
                    "share_of_step": float(ms_v[dom] / max(ms_k.sum(), 1e-9))}
    else:
        roofline = hbm_entry(dom)
    # the join-class kernels that move HBM data in this step (M_{t+1} producers, table writer)
    hbm_kernels = {gsi.KVARIANT[i]: hbm_entry(i) for i in range(nv)
                   if launches_v[i] and gsi.KVARIANT[i] in ("next_lean", "join_next", "final_table", "join_table")}
    roofline.update({
        "per_variant": {gsi.KVARIANT[i]: {"ms": float(ms_v[i]), "launches": int(launches_v[i]),
                                          "alg_GB": float(bytes_v[i] / 1e9), "items": int(items_v[i]),
                                          "frac": float(bytes_v[i] / (ms_v[i] / 1e3) / 1e9 / peak) if ms_v[i] else 0.0}
                        for i in range(nv) if launches_v[i]},
        "hbm_kernels": hbm_kernels,
        "per_class_ms": {gsi.KCLASS[i]: float(ms_k[i]) for i in range(6)},
        "model": "hbm kernels: algorithmic bytes = what the kernel must move at least once: rows it extends "
                 "(row, loc, F), candidates streamed from ci (shared N(v,l0)∩C(u) runs are L2-resident, not "
                 "charged per slot), one 32 B PCSR sector + fpos per lookup, every byte written; alu: ALU-pipe "
                 "lane-ops of the fingerprint spec per match (DESIGN.md §6)"})

    # ---- multi-GPU balance, emulated on this GPU: each rank's shard run alone -------------
    balance = None
    if ws == 1 and not args.no_balance:
        balance = {}
        for W_ in (2, 4, 8):
            per_rank = []
            tot = 0
            for r_ in range(W_):
                t_ms, c_ = timed(lambda: step(HEAD, timeout=args.enum_timeout,
                                              sh=dict(shard_rank=r_, shard_count=W_, shard_pieces=args.shard_pieces)))
                per_rank.append(t_ms)
                tot += int(c_.sum().item())
            balance[str(W_)] = {"rank_ms": per_rank, "max_ms": max(per_rank),
                                "efficiency": sum(per_rank) / (W_ * max(per_rank)),
                                "count_equal": tot == total_matches}

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        import oracle
        t = time.time()
        og = oracle.OracleGraph(g)
        threads = len(os.sched_getaffinity(0))
        m, s, d, to = oracle_sample(og, qs, args.cpu_budget, args.ref_query_timeout, threads)
        cpu = {"value": m / s if s > 0 else 0.0, "unit": "matches/s", "cores": threads, "kind": "oracle",
               "sample": f"first {d} queries of the batch, per-query timeout {args.ref_query_timeout}s "
                         f"({to} timed out, partial counts kept); {s:.1f}s of CPU work",
               "ms_per_query": 1000.0 * s / max(d, 1)}
        log(f"[bench] oracle baseline {time.time() - t:.1f}s incl. index build")

    line = {
        "metric": "matches/s", "value": value, "unit": "matches/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": workload_config(args, g),
        "ms_per_query": ms_per_step / len(qs), "matches_per_step": total_matches,
        "query_ms_p50": float(np.percentile(q_ms, 50)), "query_ms_p95": float(np.percentile(q_ms, 95)),
        "per_query": [{"count": int(c), "ms": round(float(t_), 3)} for c, t_ in zip(per_query_counts, q_ms_by_query)],
        "capped_queries_per_step": capped, "query_timeout_s": args.enum_timeout,
        "e2e": {"value": m_e2e * args.steps / e2e_s, "unit": "matches/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_query": 1000.0 * e2e_s / args.steps / len(qs)},
        "kernel_variants": _variants(launch_stats), "count_only": count_only, "table": table, "roofline": roofline, "multi_gpu_balance_emulated": balance,
        "small_queries": small,
        "cpu_baseline_single_thread": cpu_single,
        "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches,
        "graph": {"n_groups": info["n_groups"], "max_chain": info["max_chain"],
                  "bytes_total": info["bytes_total"], "build_ms": info["ms_build"]},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _variants(stats):
    out = {}
    for s_ in stats:
        for k_, v_ in s_["variants"].items():
            out[k_] = out.get(k_, 0) + v_
    return out


def oracle_single_thread(nq, k, timeout_s=2.0):
    """The CPU oracle, one thread, per query on C1 (the Fig. 1 query) and the C2 / C3 walk
    queries the GPU latency section runs: median of 3 runs per query (C1) / one run (C2, C3,
    per-query timeout, partial counts kept), then p50 / mean over the queries."""
    import oracle
    out = {}
    g1, q1 = W.fig1()
    og = oracle.OracleGraph(g1)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        c, _, _ = oracle.match(og, q1, table=False, threads=1)
        ts.append(1000.0 * (time.perf_counter() - t))
    out["C1"] = {"queries": 1, "p50_ms": float(np.median(ts)), "matches": int(c)}
    for cfg in ("C2", "C3"):
        g, qs = make_workload(cfg, nq, k, "cuda" if _cuda_ok() else "cpu")   # the GPU section's inputs
        og = oracle.OracleGraph(g)
        per, tot, touts = [], 0, 0
        for q in qs:
            t = time.perf_counter()
            c, _, _ = oracle.match(og, q, table=False, threads=1, timeout=timeout_s, partial=True)
            el = 1000.0 * (time.perf_counter() - t)
            touts += el >= 1000.0 * timeout_s
            per.append(el)
            tot += c
        a = np.array(per)
        out[cfg] = {"queries": len(per), "p50_ms": float(np.percentile(a, 50)), "mean_ms": float(a.mean()),
                    "p95_ms": float(np.percentile(a, 95)), "timeouts": int(touts), "matches": int(tot)}
    out["threads"] = 1
    out["note"] = "oracle/ backtracker as it stands, one host thread, per-query wall time; a baseline, not the target"
    return out


def small_query_latency(gsi, cfg, nq, k, device):
    """Latency of single queries on a small-query config: each of the nq walk queries runs
    alone (prepared, count-only) 5 times after one warm-up; per query the median of the host
    wall time around the synchronous gsi_query_run (filter, plan, every level, count on the
    host), then p50 / mean / p95 over the queries, with the kernel path taken."""
    import torch
    g, qs = make_workload(cfg, nq, k, "cuda")
    graph = gsi.build(g, device=device)
    torch.cuda.synchronize()
    prepared = [gsi.prepare(graph, q) for q in qs]
    per_q, dev_ms, paths, counts = [], [], {}, []
    for p in prepared:
        gsi.gsi_query_run(graph, p, fingerprint=False)
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            r = gsi.gsi_query_run(graph, p, fingerprint=False)
            ts.append(1000.0 * (time.perf_counter() - t))
        st = r.stats()
        per_q.append(float(np.median(ts)))
        dev_ms.append(st["ms_total"])
        counts.append(r.count)
        path = "small" if st["variants"].get("small", 0) and not st["small_aborted"] else "regular"
        paths[path] = paths.get(path, 0) + 1
    a = np.array(per_q)
    out = {"workload": BENCH_CONFIGS[cfg]["desc"], "queries": len(per_q), "p50_ms": float(np.percentile(a, 50)),
           "mean_ms": float(a.mean()), "p95_ms": float(np.percentile(a, 95)), "paths": paths,
           "matches": int(sum(counts)), "timing": "host wall time around one synchronous gsi_query_run "
                                                 "(prepared query, count-only), median of 5 per query"}
    del prepared, graph
    gsi.gsi_trim_workspace(device)
    torch.cuda.empty_cache()
    return out


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks of this script (one per GPU,
    NCCL over 127.0.0.1) and return their exit status."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"[bench] --gpus {args.gpus} but only {have} CUDA device(s) visible")
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gsi", "reference"], default="gsi")
    ap.add_argument("--config", choices=sorted(BENCH_CONFIGS), default="C5m")
    ap.add_argument("--scale", type=int, default=None, help="override the R-MAT scale (C5 only)")
    ap.add_argument("--queries", type=int, default=16)
    ap.add_argument("--k", type=int, default=12)
    ap.add_argument("--query-timeout", type=float, default=1.0,
                    help="per-query cap; a capped query reports the exact count of its completed prefix")
    ap.add_argument("--ref-query-timeout", type=float, default=5.0)
    ap.add_argument("--ref-step-budget", type=float, default=8.0)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["fp", "count", "table"], default="fp",
                    help="headline pass: fp = every match produced, read and hashed (default); count = the "
                         "closed-form count path")
    ap.add_argument("--no-count-only", action="store_true", help="skip the secondary count-only pass")
    ap.add_argument("--concurrency", type=int, default=2, help="queries in flight (host workers / streams)")
    ap.add_argument("--enum-timeout", type=float, default=30.0, help="per-query cap of the headline and table passes")
    ap.add_argument("--no-table", action="store_true", help="skip the with-table pass")
    ap.add_argument("--table-max-gb", type=float, default=32.0, help="table pass: queries whose table fits")
    ap.add_argument("--no-balance", action="store_true", help="skip the emulated multi-GPU balance")
    ap.add_argument("--shard-pieces", type=int, default=8, help="interleaved shard pieces per rank (N > 1)")
    ap.add_argument("--no-small", action="store_true", help="skip the small-query latency section")
    ap.add_argument("--small-configs", nargs="*", default=["C2", "C3", "C4"])
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if args.impl == "gsi" and ws != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={ws}")
        sys.exit(1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gsi(args)


if __name__ == "__main__":
    main()
