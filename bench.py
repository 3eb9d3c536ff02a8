#!/usr/bin/env python
"""PQTopK hot-path benchmark (B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step is one pass of the whole hot path over one batch: K1 sub-id scores
(pq_subscores) -> K2 fused gather-sum-select -> K3 merge (pq_score_topk) for
batches, ONE fused launch (pq_search: K7, or K6 for long streams) for B <= 4,
and for N > 1 GPUs (item-sharded catalogue) an NCCL all-gather of the B x K
local results followed by pq_merge_topk.  Metric (BASELINE.json): user-item
scores/s = B * N_items / step time (whole job), plus top-K queries/s.

Timing: W untimed warm-up steps; K timed steps bracketed by barrier +
synchronize; each step timed with CUDA events on the launching stream; before
each step a 256 MiB buffer is written (L2 flush, outside the events); the
reported time is the max over ranks.  The roofline block uses the fused
kernel's own launch time (events recorded by the library around K2).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import pqsynth  # noqa: E402

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(FALLBACK_PEAKS)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, torch_dev: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(torch_dev).uuid)
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hh = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hh)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        h = hh
            except Exception:
                h = None
            if h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                ids = [int(x) for x in vis.split(",") if x.strip().isdigit()]
                h = pynvml.nvmlDeviceGetHandleByIndex(ids[torch_dev] if torch_dev < len(ids) else torch_dev)
            self.h = h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def launched_by_torchrun() -> bool:
    """Under torch.distributed.run (WORLD_SIZE set) the sharded path runs --
    process group, packed all-gather and merge -- even at world size 1."""
    return "WORLD_SIZE" in os.environ


def parity_users(B: int, n: int = 64):
    """Users checked against the oracle: n users spread evenly over the batch
    (stride B/n), so every user group / CTA tile of the batch is sampled."""
    n = min(n, B)
    return sorted({(j * B) // n for j in range(n)})


def shard(N, world, rank):
    from paper_2408_09992_b200.dist import shard_range
    return shard_range(N, world, rank)


def workload_name(cfg):
    return (f"{cfg.name}: N={cfg.N:,} m={cfg.m} b={cfg.b} d={cfg.d} B={cfg.B} K={cfg.K} "
            f"codes={cfg.codes}")


def oracle_all_cores():
    """The oracle on every host core this process may use (torchrun exports
    OMP_NUM_THREADS=1 to its ranks; the CPU baseline wants the whole host)."""
    import oracle
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:                           # pragma: no cover - non-Linux
        n = os.cpu_count() or 1
    oracle.set_threads(n)
    return oracle


def cpu_oracle_sample(cfg, codes, S_host, gpu_ids, gpu_sc, budget_s=12.0, max_users=64):
    """Time the CPU oracle (Alg. 1, plain C + OpenMP) on a bounded sample of
    users over the full catalogue -- users spread over the whole batch
    (parity_users) -- and check those users bit-exactly against the GPU result.
    Also times one user with ONE thread (the per-core figure)."""
    oracle = oracle_all_cores()
    users = parity_users(cfg.B, max_users)
    done, t_tot, exact, checked = 0, 0.0, 0, []
    for u in users:
        if t_tot >= budget_s:
            break
        t0 = time.perf_counter()
        ids, sc = oracle.pq_topk(codes, S_host[u:u + 1], cfg.K)
        t_tot += time.perf_counter() - t0
        if gpu_ids is not None:
            exact += int(np.array_equal(ids[0], gpu_ids[u]) and
                         np.array_equal(sc[0].view(np.uint32), gpu_sc[u].view(np.uint32)))
        checked.append(u)
        done += 1
    cores = oracle.max_threads()
    # one thread, one user (bounded: about 2e9 lookups, ~1 s)
    n1 = min(cfg.N, max(1, int(2e9 // max(cfg.m, 1))))
    oracle.set_threads(1)
    try:
        t0 = time.perf_counter()
        oracle.pq_topk(codes[:n1], S_host[:1], cfg.K)
        t1 = time.perf_counter() - t0
    finally:
        oracle.set_threads(cores)
    stride = (cfg.B // len(users)) if users else 0
    desc = (f"users {checked[0]}..{checked[-1]} step {stride} ({done} of {cfg.B})" if done > 1
            else f"user {checked[0]} of {cfg.B}")
    cpu = {"value": done * cfg.N / t_tot, "unit": "user-item scores/s", "cores": cores,
           "kind": "oracle", "cpu_model": oracle.cpu_model(),
           "sample": f"{desc} over all {cfg.N:,} items (Alg. 1 item-major, fp32 k-ordered sums, "
                     f"heap top-K), {t_tot:.1f} s",
           "one_thread": {"value": n1 / t1, "unit": "user-item scores/s",
                          "sample": f"user 0 over items 0..{n1 - 1:,}, 1 thread, {t1:.2f} s"}}
    return cpu, checked, exact


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    oracle = oracle_all_cores()
    cfg = pqsynth.CONFIGS[args.config]
    codes = pqsynth.codes(cfg)
    P = pqsynth.psi(cfg)
    F = pqsynth.phi(cfg)
    # users per step: about 1 s of oracle work per step at ~1e9 lookups/s/core
    lk = cfg.N * cfg.m
    upstep = max(1, min(cfg.B, int(1.5e9 * oracle.max_threads() / max(lk, 1) / 4)))
    S_all = None
    times = []
    for s in range(args.warmup + args.steps):
        u0 = (s * upstep) % cfg.B
        Fu = F[u0:u0 + upstep]
        t0 = time.perf_counter()
        S = oracle.subscores(Fu, P)                # Eq. 4 (fp64 -> fp32)
        oracle.pq_topk(codes, S, cfg.K)            # Alg. 1 + TopK
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
        S_all = S
    del S_all
    t = sum(times) / len(times)
    value = upstep * cfg.N / t
    line = {
        "impl": "reference", "metric": "user-item scores/s", "value": value, "unit": "user-item scores/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (pqsynth, seeded)",
        "config": {"workload": workload_name(cfg), "users_per_step": upstep},
        "cpu_baseline": {"value": value, "unit": "user-item scores/s", "cores": oracle.max_threads(),
                         "kind": "oracle",
                         "sample": f"{upstep} user(s) per step over all {cfg.N:,} items (K1 fp64 + Alg. 1)"},
        "e2e": {"value": value, "unit": "user-item scores/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "queries_per_s": upstep / t,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- baselines
def compare_paths(pq, torch, idx, cfg, F_d, P_d, S, step, flush, pq_ms, reps=3):
    """The paper's comparison methods on the same batch, on the GPU:
    dense scoring r = W phi (Eq. 2-3; W reconstructed once, outside the timing; fp32
    SGEMM + top-K) and RecJPQScore (Alg. 2: split-major accumulation over an
    N-length score array + top-K, with K1).  Speed-ups against the PQTopK step."""
    K = cfg.K
    W = pq.pq_reconstruct(idx, P_d)
    torch.cuda.synchronize()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    dws = torch.empty(max(1, int(pq.load_library().pq_dense_workspace_bytes(cfg.N, cfg.B, K))),
                      dtype=torch.uint8, device=S.device)
    rws = torch.empty(max(1, idx.recjpq_workspace_bytes(cfg.B, K)), dtype=torch.uint8, device=S.device)
    dense_ms = timed(lambda: pq.pq_dense_topk(W, F_d, K, ws=dws))
    recjpq_ms = timed(lambda: (pq.pq_subscores(F_d, P_d, S), pq.pq_recjpq_topk(idx, S, K, ws=rws)))
    del W
    return {"pq_ms": pq_ms, "dense_ms": dense_ms, "recjpq_ms": recjpq_ms,
            "speedup_vs_dense": dense_ms / pq_ms, "speedup_vs_recjpq": recjpq_ms / pq_ms,
            "dense": "W = reconstruct (Eq. 2) resident; fp32 SGEMM (no TF32) + exact top-K",
            "recjpq": "K1 + Alg. 2 (split-major fp32 accumulator in HBM) + exact top-K",
            "paper_cpu_context": "4.5x vs SASRec dense, 1.56x vs RecJPQ (Ryzen 5950X, TF 2.11, Gowalla "
                                 "~1.3M items, total mRT incl. backbone; BASELINE.md)"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2408_09992_b200 as pq

    world, rank, local = dist_env()
    sharded = launched_by_torchrun()
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only "
                         f"{torch.cuda.device_count()} GPU(s) are visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if sharded:
        dist.init_process_group("nccl", device_id=dev)
    pq.load_library()
    cfg = pqsynth.CONFIGS[args.config]
    B, K, m, b, d = cfg.B, cfg.K, cfg.m, cfg.b, cfg.d
    lo, hi = shard(cfg.N, world, rank)
    n_local = hi - lo
    if n_local <= 0:
        raise SystemExit(f"bench.py: {cfg.name} has fewer items ({cfg.N}) than ranks ({world})")

    codes = pqsynth.codes(cfg, lo, hi)
    P = pqsynth.psi(cfg)
    F = pqsynth.phi(cfg)

    t0 = time.perf_counter()
    # every config builds the colour-paired layout on the GPU (the batched K2 v3
    # rows; for B <= 4 the paired row-order codes of K6 / K7)
    idx = pq.pq_create(codes, b=b, id_base=lo)
    torch.cuda.synchronize()
    create_s = time.perf_counter() - t0
    if args.variant or args.tuning:
        tun = dict(kv.split("=") for kv in args.tuning.split(",") if kv) if args.tuning else {}
        tun = {k: int(v) for k, v in tun.items()}
        if args.variant:
            tun["variant"] = args.variant
        idx.set_tuning(**tun)
    # B <= 4 (the serving case): pq_search runs the whole path as ONE fused
    # kernel (K7 with chunk-resident codes, else K6 with a streamed code ring:
    # sub-id scores + gather-sum + select + merge); that call is the step
    fused = args.fused == "on" and idx.search_plan(B, d, K)["variant"] in (5, 7)
    plan = idx.search_plan(B, d, K) if fused else idx.plan(B, K)
    layout = idx.layout()

    from paper_2408_09992_b200.dist import alloc_local, gather_merge

    F_d = torch.from_numpy(F).to(dev)
    P_d = torch.from_numpy(P).to(dev)
    S = torch.empty((B, m, b), dtype=torch.float32, device=dev)
    # the local result is written straight into the packed [2][B][K] buffer the
    # all-gather sends (plane 0 ids, plane 1 score bits)
    packed, ids, sc = alloc_local(B, K, dev)
    ws = torch.empty(idx.topk_workspace_bytes(B, K), dtype=torch.uint8, device=dev)
    sws = torch.empty(idx.search_workspace_bytes(B, d, K), dtype=torch.uint8, device=dev)
    if sharded:
        out_ids = torch.empty((B, K), dtype=torch.int32, device=dev)
        out_sc = torch.empty((B, K), dtype=torch.float32, device=dev)
        gbuf = torch.empty((world * 2, B, K), dtype=torch.int32, device=dev)
        mws_n = int(pq.load_library().pq_merge_workspace_bytes(world, B, K))
        mws = torch.empty(max(mws_n, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if args.no_flush:                                # diagnostics only: the line is marked invalid
        flush = torch.empty(0, dtype=torch.uint8, device=dev)

    def exchange():
        # ONE NCCL all-gather of the packed B x K (id, score) pairs + pq_merge_topk_packed (dist.py)
        gather_merge(packed, out=(out_ids, out_sc), ws=mws, gathered=gbuf)

    def step():
        if fused:
            pq.pq_search(idx, F_d, P_d, K, ws=sws, ids=ids, scores=sc)
        else:
            pq.pq_subscores(F_d, P_d, S)
            pq.pq_score_topk(idx, S, K, ws=ws, ids=ids, scores=sc)
        if sharded:
            exchange()

    def barrier():
        if sharded:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ------------------------------------------------------------- timed (device-resident)
    # The step is captured once into a CUDA graph and replayed (single GPU;
    # removes host launch gaps, which dominate the small configs).  The fused
    # kernel's own launch time for the roofline is measured in a separate
    # non-graph pass with the library's per-launch events.
    use_graph = args.graph == "on" or (args.graph == "auto" and not sharded)
    graph = None
    if use_graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        n_cap0 = pq.launch_count()
        with torch.cuda.graph(graph):
            step()
        launches_per_step = pq.launch_count() - n_cap0
        for _ in range(max(1, args.warmup)):          # warm the graph replay path too
            graph.replay()
        torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    n_launch0 = pq.launch_count()
    with sampler:
        barrier()
        torch.cuda.synchronize()
        # the GPU idles ~2 ms while the host enqueues every timed step, so a host
        # hiccup (GIL, sampler thread) can never open a gap inside a timed step
        torch.cuda._sleep(4_000_000)
        for e0, e1 in evs:
            flush.fill_(1)
            e0.record()
            if graph is not None:
                graph.replay()
            else:
                step()
            e1.record()
        torch.cuda.synchronize()
        barrier()
    gpu_launches = (launches_per_step * args.steps) if graph is not None else pq.launch_count() - n_launch0
    step_ms = [a.elapsed_time(c) for a, c in evs]
    tot_ms = sum(step_ms)
    # supplementary (not the bench value): the same step with a warm L2 when the
    # codes fit in it (SURVEY §8(d) L2 policy: report warm and cold)
    warm_ms = None
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    if not sharded and n_local * m < l2_bytes:
        evw = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for e0, e1 in evw:
            e0.record()
            if graph is not None:
                graph.replay()
            else:
                step()
            e1.record()
        torch.cuda.synchronize()
        warm_ms = statistics.median([a.elapsed_time(c) for a, c in evw])
    # fused-kernel launch time (library events around K2), outside the graph
    idx.timing_enable(True)
    idx.timing_read()
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    k2_ms, k3_ms, n_k2 = idx.timing_read()
    idx.timing_enable(False)
    t = torch.tensor([tot_ms, k2_ms], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms_max, k2_ms_max = float(t[0]), float(t[1])
    ms_per_step = tot_ms_max / args.steps
    value = B * cfg.N / (ms_per_step / 1e3)

    # ------------------------------------------------------------- e2e (host buffers)
    # Per step: the batch's sequence embeddings phi from pinned host memory in, the
    # top-K ids/scores back to pinned host memory, through the public whole-step
    # call (pq_search).  The sub-item embeddings Psi are model weights that live
    # on the device with the index (like the codes), not per-query inputs.
    F_h = torch.from_numpy(F).pin_memory()
    ids_h = torch.empty((B, K), dtype=torch.int32).pin_memory()
    sc_h = torch.empty((B, K), dtype=torch.float32).pin_memory()

    def e2e_step():
        if not sharded:
            pq.pq_search(idx, F_h, P_d, K, ws=sws, ids=ids_h, scores=sc_h)
        else:                                        # host inputs -> local result -> exchange -> host
            pq.pq_search(idx, F_h, P_d, K, ws=sws, ids=ids, scores=sc)
            exchange()
            ids_h.copy_(out_ids, non_blocking=True)
            sc_h.copy_(out_sc, non_blocking=True)
    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    evs2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    barrier()
    for e0, e1 in evs2:
        flush.fill_(1)
        e0.record()
        e2e_step()
        e1.record()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = sum(a.elapsed_time(c) for a, c in evs2)
    t2 = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = B * cfg.N / (float(t2[0]) / args.steps / 1e3)

    # final results for parity sampling (rank 0 at N = 1); the fused kernel's own S
    if fused:
        pq.pq_search(idx, F_d, P_d, K, ws=sws, ids=ids, scores=sc, S_out=S)
        if sharded:
            exchange()
    torch.cuda.synchronize()
    res_ids = (out_ids if sharded else ids).cpu().numpy()
    res_sc = (out_sc if sharded else sc).cpu().numpy()

    if rank != 0:
        if sharded:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk = peaks()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = float(pk.get("sm_max_mhz", 1965.0))
    peak_lookups = nsm * 32 * f_max * 1e6            # 32 four-byte smem lookups / clk / SM
    k2_avg_s = (k2_ms_max / max(n_k2, 1)) / 1e3
    lookups = B * n_local * m                        # algorithmic lookups per K2 launch
    achieved = lookups / k2_avg_s
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"k2_traffic_{cfg.name}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    # The binding roofline of the fused kernel: the shared-memory lookup rate
    # (m lookups per user-item pair) or, for tiny batches, the HBM stream of
    # the code matrix (m bytes per item, once per batch) -- whichever takes longer.
    hbm_bytes = n_local * m + B * m * b * 4 + B * K * 8          # algorithmic bytes per launch
    if fused:                                        # K6 reads phi and Psi instead of S
        hbm_bytes = n_local * m + B * d * 4 + b * d * 4 + B * K * 8
    peak_hbm = pk["hbm_gbs"] * 1e9
    t_smem, t_hbm = lookups / peak_lookups, hbm_bytes / peak_hbm
    kname = {1: "k2_score_select (v1 row groups)",
             3: "k2_tiled (v3: fused gather-sum-select, 4 users/lane)",
             4: "k2_latency (v4: small-batch fused gather-sum-select)",
             5: "k6_query (K1 + gather-sum + select + merge in one launch, B <= 4; streamed code ring)",
             7: "k7_resident (K1 + gather-sum + select + merge in one launch, B <= 4; chunk-resident codes)"
             }.get(plan["variant"], "k2")
    common = {
        "kernel": kname, "traffic": traffic,
        "per_launch": {"lookups": lookups, "algorithmic_hbm_bytes": hbm_bytes, "k2_ms": k2_avg_s * 1e3},
        "k2_share_of_step": k2_avg_s * 1e3 / ms_per_step,
        "smem_frac": achieved / peak_lookups,
        # exact first-pair tables (b = 16): the kernel performs m - 1 lookups per pair
        "lookups_executed_per_pair": (m - 1) if (plan["variant"] == 3 and b == 16 and m in (4, 8)) else m,
        "smem_frac_executed": achieved / peak_lookups *
            (((m - 1) / m) if (plan["variant"] == 3 and b == 16 and m in (4, 8)) else 1.0),
        "hbm_frac_algorithmic": (hbm_bytes / k2_avg_s) / peak_hbm,
        "peak_source_smem": f"{nsm} SMs x 32 banks x 4 B x {f_max:.0f} MHz (sm_max_mhz, {pk['source']}); "
                            "128 B/clk/SM attained by the paired LDS.128 pattern in the smem microbenchmark "
                            "(profiles/r01/ubench/smem_rate_b200.txt)",
        "peak_source_hbm": f"hbm_gbs {pk['hbm_gbs']} ({pk['source']})",
    }
    if t_smem >= t_hbm:
        roofline = {"bound": "smem", "achieved": achieved / 1e9, "peak": peak_lookups / 1e9,
                    "unit": "G lookups/s", "frac": achieved / peak_lookups, **common}
    else:
        roofline = {"bound": "hbm", "achieved": hbm_bytes / k2_avg_s / 1e9, "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": (hbm_bytes / k2_avg_s) / peak_hbm, **common}
    cpu = None
    parity = None
    if not args.no_cpu_baseline:
        # rank 0 checks the MERGED global result against the oracle over the
        # WHOLE catalogue (at N > 1 it regenerates the other shards' codes)
        full_codes = codes if world == 1 else pqsynth.codes(cfg)
        cpu, users, nexact = cpu_oracle_sample(cfg, full_codes, S.cpu().numpy(), res_ids, res_sc)
        del full_codes
        parity = (f"bit-exact vs oracle (given GPU S) on {nexact}/{len(users)} sampled users "
                  f"(users {users[0]}..{users[-1]}, stride {cfg.B // max(1, len(parity_users(cfg.B)))}"
                  f"{', merged over ' + str(world) + ' shards' if sharded else ''})")
    clocks = sampler.summary()
    comparison = None
    want_cmp = args.compare == "on" or (args.compare == "auto" and cfg.name in ("c2", "c3"))
    if not sharded and want_cmp and cfg.N * d * 4 <= (48 << 30):
        comparison = compare_paths(pq, torch, idx, cfg, F_d, P_d, S, step, flush, ms_per_step)
    line = {
        "metric": "user-item scores/s", "value": value, "unit": "user-item scores/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (pqsynth, seeded; BASELINE.json config recipe)",
        "config": {"workload": workload_name(cfg), "items_per_gpu": n_local,
                   "k2_plan": plan, "layout": layout,
                   "parallelism": (f"item-shard x{world} (NCCL all-gather of packed B x K pairs + "
                                   "pq_merge_topk_packed)") if sharded else "single GPU",
                   "cuda_graph": graph is not None,
                   "l2": ("NO L2 flush (diagnostic run, not a bench value)" if args.no_flush else
                          "256 MiB L2 flush before every timed step (outside events)")},
        "queries_per_s": B / (ms_per_step / 1e3),
        "e2e": {"value": e2e_value, "unit": "user-item scores/s",
                "h2d_bytes_per_step": B * d * 4,
                "path": "pq_search: phi pinned host -> device, top-K ids/scores device -> pinned host, every "
                        "step; Psi (model weights) and the codes resident with the index",
                "d2h_bytes_per_step": B * K * 8},
        "gpu_launches": gpu_launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "parity": parity,
        "clocks": clocks,
        "create_s": create_s,
        "comparison": comparison,
        "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms),
                    "p10": float(np.percentile(step_ms, 10)), "p90": float(np.percentile(step_ms, 90)),
                    "warm_l2_median": warm_ms},
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_torchrun(n: int) -> int:
    import socket
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(pqsynth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--compare", default="auto", choices=["auto", "on", "off"],
                    help="time the paper's baselines beside PQTopK (auto: c2, c3)")
    ap.add_argument("--variant", type=int, default=0,
                    help="force the K2 variant (1 row groups, 3 tiled, 4 small batch; 5 = fused K6 / 7 = fused K7 in pq_search; 0 = auto)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: single GPU)")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics: skip the L2 flush (not a valid bench line)")
    ap.add_argument("--fused", default="on", choices=["on", "off"],
                    help="B <= 4: run pq_search's single-launch K6 kernel (off: K1 + K2 v4 + K3)")
    ap.add_argument("--tuning", default="", help="K2 launch tuning, e.g. warps=8,chunks=9 (diagnostics)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if launched_by_torchrun():
        ws_env = int(os.environ["WORLD_SIZE"])
        if ws_env != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}; "
                             "launch one rank per GPU (torch.distributed.run --nproc-per-node N)")
    elif args.gpus > 1 and args.impl == "ours":
        # not under torchrun: re-launch this command as N ranks, one per GPU
        sys.exit(relaunch_torchrun(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
