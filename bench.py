"""bench.py — throughput of the region-streaming hot path (BASELINE.json metric:
"input items/sec and SIMD lane occupancy vs region length, signal vs tagged,
1-8 B200").

Default (N=1): BASELINE configs[1], region-length sweep, in the fixed-children
reading of SURVEY §8(d): N = 2^29 int32 children (the paper's 512M integers,
P:565-567), fixed region length L = 4096 (R = 131072), 3 HASH_LT filters,
SUM_I64, signal strategy.  A "step" is one rs_pipeline_run over that batch
(enumerate -> 3 filters -> aggregate, all §8(a) rows).  Inputs (2 GB) exceed
the 126 MB L2, so no flush is needed between steps.

--impl reference times the CPU oracle (the paper-derived interpreter) on the
host cores instead (the tier's reference arm).
Under torchrun (N>1) every rank runs its own shard (whole regions, weak
scaling) and the per-region aggregates are gathered to rank 0 with NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input items/sec and SIMD lane occupancy vs region length, signal vs tagged, 1-8 B200"
FALLBACK_HBM_GBS = 6650.0        # /opt/skills/guides/B200_PROFILING.md fallback ("of fallback")


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            for k in ("hbm_gbs", "hbm_GBps", "hbm"):
                if k in d:
                    v = d[k]
                    return float(v["value"] if isinstance(v, dict) else v), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        self.t_on = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([time.time()] + [x.strip() for x in line.split(",")])

    def wait_ready(self, timeout=5.0):
        """Block until the sampler delivers its first sample (nvidia-smi start-up)."""
        t0 = time.time()
        while self.proc and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.05)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        # samples inside the timed window (100 ms sampling; short windows take the
        # nearest samples within +-0.25 s)
        win = getattr(self, "window", None)
        smp = self.samples
        if win:
            inside = [s for s in smp if win[0] <= s[0] <= win[1]]
            smp = inside or [s for s in smp if win[0] - 0.25 <= s[0] <= win[1] + 0.25]
        if not smp:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in smp if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in smp if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in smp:
            for n, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(smp)}


# ------------------------------------------------------------------ workloads
def workload_spec(name):
    import synth
    if name == "sweep_fixed_L4096":
        return dict(N=1 << 29, dist="fixed", L=4096, stages=synth.sweep_stages(3), agg="sum_i64", dtype="i32")
    if name.startswith("sweep_"):
        # sweep_<fixed|var>_L<L>
        _, dist, l = name.split("_")
        return dict(N=1 << 29, dist=dist, L=int(l[1:]), stages=synth.sweep_stages(3), agg="sum_i64", dtype="i32")
    if name == "zipf":
        return dict(N=1 << 30, dist="zipf", L=0, stages=synth.sweep_stages(3), agg="sum_i64", dtype="i32")
    if name == "graph":
        return dict(N=16 << 24, dist="rmat", L=0, stages=[("lt_u32", 1 << 31)], agg="count_min_u32", dtype="u32")
    if name == "text":
        return dict(N=1 << 32, dist="text", L=0, stages=synth.text_stages(), agg="count_xor64", dtype="u8")
    raise ValueError(name)


def make_inputs(spec, seed, device):
    import synth
    import torch
    N, dist, L = spec["N"], spec["dist"], spec["L"]
    if dist == "rmat":
        return synth.torch_rmat_csr(24, 16, seed=seed, device=device)
    if dist == "text":
        return synth.torch_text(N, seed=seed, device=device)
    if dist == "fixed":
        lens = torch.full((N // L,), L, dtype=torch.int64, device=device)
    elif dist == "var":
        lens = synth.torch_lengths(N // L, "var", L=L, seed=seed, device=device)
    else:
        lens = synth.torch_lengths(int(N / 208.7), "zipf", seed=seed, device=device)
    off = synth.torch_offsets(lens)
    n = int(off[-1].item())
    vals = synth.torch_values(n, spec["dtype"], seed=seed + 1, device=device)
    return vals, off


def alg_bytes(n, R, agg):
    """Payload read once + offsets read once + one aggregate written per region
    (SURVEY §8(d))."""
    out_b = {"sum_i64": 8, "sum_f32": 4, "count_min_u32": 8, "count_xor64": 16}[agg]
    esz = 1 if agg == "count_xor64" else 4
    return esz * n + 8 * (R + 1) + out_b * R


# ------------------------------------------------------------------- oracle
def oracle_rate(vals_h, off_h, stages, agg, budget_s=10.0, cores=None):
    """Time the CPU oracle's pipeline interpreter (as it stands) on a bounded
    prefix sample of the workload, sharded over host cores by whole regions
    (regions are independent contexts; ctypes releases the GIL)."""
    import concurrent.futures as cf

    import oracle
    cores = cores or len(os.sched_getaffinity(0))
    R = off_h.size - 1
    # calibrate on a small sample to size a ~budget_s run
    r_small = min(R, max(1, int(np.searchsorted(off_h, off_h[0] + (1 << 18)))))
    t0 = time.perf_counter()
    oracle.interp(vals_h, off_h[:r_small + 1], stages, agg, check=False)
    dt = time.perf_counter() - t0
    n_small = int(off_h[r_small] - off_h[0])
    per_item = dt / max(1, n_small)
    target = int(budget_s * cores / max(per_item, 1e-12))
    r_end = int(min(R, max(cores, np.searchsorted(off_h, off_h[0] + target))))
    bounds = np.linspace(0, r_end, cores + 1).astype(np.int64)

    def work(i):
        a, b = int(bounds[i]), int(bounds[i + 1])
        if b > a:
            oracle.interp(vals_h, off_h[a:b + 1], stages, agg, check=False)
        return int(off_h[b] - off_h[a])

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(cores) as ex:
        items = sum(ex.map(work, range(cores)))
    wall = time.perf_counter() - t0
    return items / wall, cores, f"interpreter on regions [0,{r_end}) = {items} children, {cores} threads, {wall:.1f}s"


def _prefix(off_h, n_items):
    """Regions [0, r) covering about n_items children from the stream start."""
    return int(min(off_h.size - 1, max(1, np.searchsorted(off_h, off_h[0] + n_items))))


def _rate_1t(fn, vals_h, off_h, budget_s):
    """Children/s of fn(vals, off) on one thread over a prefix sized for ~budget_s."""
    r = _prefix(off_h, 1 << 16)
    t0 = time.perf_counter()
    fn(vals_h, off_h[:r + 1])
    per = (time.perf_counter() - t0) / max(1, int(off_h[r] - off_h[0]))
    r = _prefix(off_h, int(budget_s / max(per, 1e-12)))
    t0 = time.perf_counter()
    fn(vals_h, off_h[:r + 1])
    dt = time.perf_counter() - t0
    n = int(off_h[r] - off_h[0])
    return n / dt, f"regions [0,{r}) = {n} children in {dt:.1f}s"


def cpu_baseline(vals_h, off_h, spec, budget_s=10.0):
    """The oracle as it stands on this box's host cores:
    (i) plain fold, 1 thread; (ii) interpreter, 1 thread; (iii) interpreter
    on all cores, one instance per contiguous region shard -- the value."""
    import oracle
    st, agg = spec["stages"], spec["agg"]
    b1, bd = _rate_1t(lambda v, o: oracle.brute(v, o, st, agg), vals_h, off_h, budget_s / 4)
    i1, idesc = _rate_1t(lambda v, o: oracle.interp(v, o, st, agg, check=False), vals_h, off_h, budget_s / 4)
    rate, cores, desc = oracle_rate(vals_h, off_h, st, agg, budget_s=budget_s)
    return {"value": rate, "unit": "items/s", "cores": cores, "kind": "oracle", "sample": desc,
            "brute_1thread": {"value": b1, "sample": bd}, "interp_1thread": {"value": i1, "sample": idesc}}


def run_reference(args):
    """--impl reference: the CPU oracle on this box's cores (tier reference arm),
    on the same workload and seed as the GPU arm (a bounded prefix sample per step)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec = workload_spec(args.workload)
    same = True
    try:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no GPU")
        vals, off = make_inputs(spec, seed=0x5EED + 2, device=torch.device("cuda", 0))
        # the bounded sample: a prefix of up to ~2^28 children of the very same stream
        # (each step times the interpreter on as much of it as ~20 s / steps allows)
        r = _prefix(off.cpu().numpy(), 1 << 28)
        oh = off[:r + 1].cpu().numpy()
        vh = vals[: int(oh[-1])].cpu().numpy()
        del vals, off
    except Exception:
        import synth
        same = False
        n_s = 1 << 24
        if spec["dist"] == "fixed":
            lens = np.full(n_s // spec["L"], spec["L"], np.int64)
        elif spec["dist"] == "var":
            lens = synth.lengths(n_s // spec["L"], "var", L=spec["L"], seed=1)
        else:
            lens = synth.lengths(int(n_s / 208.7), "zipf", seed=1)
        oh = synth.offsets(lens)
        vh = synth.values(int(oh[-1]), spec["dtype"], seed=2)
    if spec["dtype"] == "u32":
        vh = vh.view(np.uint32)
    elif spec["dtype"] == "u8":
        vh = vh.view(np.uint8)
    rates = []
    desc = None
    cores = None
    for i in range(args.warmup + args.steps):
        r, cores, desc = oracle_rate(vh, oh, spec["stages"], spec["agg"], budget_s=max(1.0, 20.0 / max(1, args.steps)))
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    line = {"metric": METRIC, "value": v, "unit": "items/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32->int64", "data": "synthetic",
            "config": {"workload": args.workload, "strategy": "signal", "w": 128, "same_config": same,
                       "sample": "prefix of the GPU arm's stream (same generator and seed)" if same else
                       "numpy stream of the same shape"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "items/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- GPU arm
def traffic_for(workload, strategy):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(f"{workload}:{strategy}")
        except Exception:
            return None
    return None


def lane_stats(st):
    res = []
    for n in range(1, st.shape[0]):
        d, f, it, s = (int(x) for x in st[n])
        res.append({"lane_fraction": (it / (128 * d)) if d else None, "full_rate": (f / d) if d else None,
                    "ensembles": d, "items": it, "signals": s})
    return res


def _allreduce(x, op, dev, backend):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=op)
    return float(t.item())


def run_multi(args, rs, torch, dist, world, rank, local, backend):
    """N > 1 (one process per GPU): the stream is partitioned by whole regions
    (regions are independent contexts) and every rank's aggregates
    land in rank 0's dense output array at their global region offsets.

    --scaling weak (default; the driver's 1/2/4/8 run): rank k processes its
    own batch of the N=1 workload (the global stream is the concatenation of
    the ranks' batches), so per-GPU work is fixed as N grows.
    --scaling strong (BASELINE configs[4]: --workload zipf): ONE stream,
    partition() by children, rank k runs its slice through offsets into the
    shared element array (offsets[0] != 0).
    --gather peer (default): rank 0's output mapped into every rank (CUDA IPC
    over NVLink), the pipeline kernels store each region's aggregate there as
    it completes -- the gather is fused with the aggregate node and fully
    overlapped.  --gather nccl: local outputs + rs_gather_aggregates (grouped
    NCCL send/recv at exact offsets) every step."""
    from paper_2006_07478_b200.dist import RootOutputs, partition, rank_comm
    dev = torch.device("cuda", local)
    spec = workload_spec(args.workload)
    strong = args.scaling == "strong"
    if strong:
        vals, off_full = make_inputs(spec, seed=0x5EED + 2, device=dev)     # the same stream on every rank
        bounds = partition(off_full, world)
        off = off_full[bounds[rank]:bounds[rank + 1] + 1].contiguous()
        del off_full
    else:
        vals, off = make_inputs(spec, seed=0x5EED + 2 + 1000 * rank, device=dev)
        counts = [0] * world
        dist.all_gather_object(counts, int(off.numel() - 1))
        bounds = [0]
        for c in counts:
            bounds.append(bounds[-1] + c)
    R = int(off.numel() - 1)
    r_total = bounds[-1]
    n_local = int(off[-1].item() - off[0].item())
    flags = rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING
    p = rs.Pipeline(spec["stages"], spec["agg"], strategy=args.strategy, flags=flags)
    ws = p.alloc_workspace(R, vals.numel(), dev)
    ws_ptr = (ws.data_ptr() + 255) & ~255
    ws_bytes = ws.numel() - (ws_ptr - ws.data_ptr())
    stream = torch.cuda.current_stream()
    gather = args.gather if backend == "nccl" else "peer"      # NCCL needs one GPU per rank
    comm = None
    if gather == "peer":
        ro = RootOutputs(p, r_total, dev)
        o0, o1 = ro.ptrs(bounds[rank])

        def step():
            p.run_raw(vals.data_ptr(), vals.numel(), off.data_ptr(), R, o0, o1, ws_ptr, ws_bytes, stream.cuda_stream)
    else:
        comm = rank_comm()
        local_out = p.alloc_outputs(R, dev)
        root_out = p.alloc_outputs(r_total, dev) if rank == 0 else None

        def step():
            p.run(vals, off, local_out, ws)
            comm.gather(spec["agg"], local_out, bounds, root_out, root=0)

    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        clk.wait_ready()
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        w0 = time.time()
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        clk.mark(w0, time.time())
    ms = _allreduce(t0.elapsed_time(t1), dist.ReduceOp.MAX, dev, backend)
    total = _allreduce(n_local, dist.ReduceOp.SUM, dev, backend)
    main_ms = []
    for _ in range(3):
        step()
        main_ms.append(p.kernel_times()[1])
    torch.cuda.synchronize()
    dist.barrier()
    # assembled-output check: every rank's own aggregates (a fresh local run)
    # against its slice of rank 0's array, by two checksums
    chk = p.alloc_outputs(R, dev)
    p.run(vals, off, chk, ws)
    torch.cuda.synchronize()
    w = torch.arange(1, R + 1, device=dev, dtype=torch.float64)
    mine = [float(t.to(torch.float64).sum().item()) + float((t.to(torch.float64) * w).sum().item())
            for t in chk if t is not None]
    allsums = [None] * world
    dist.all_gather_object(allsums, mine)
    dist.barrier()
    ok = None
    if rank == 0:
        final = ro.out if gather == "peer" else root_out
        ok = True
        for k in range(world):
            a, b = bounds[k], bounds[k + 1]
            wk = torch.arange(1, b - a + 1, device=dev, dtype=torch.float64)
            got = [float(t[a:b].to(torch.float64).sum().item()) + float((t[a:b].to(torch.float64) * wk).sum().item())
                   for t in final if t is not None]
            ok = ok and all(abs(x - y) <= 1e-9 * max(1.0, abs(y)) for x, y in zip(got, allsums[k]))
    code = p.check()
    ms_step = ms / args.steps
    main_avg = statistics.mean(main_ms)
    peak, peak_kind = hbm_peak()
    bytes_alg = alg_bytes(n_local, R, spec["agg"])
    if rank == 0:
        line = {
            "metric": METRIC, "value": total / (ms_step / 1e3), "unit": "items/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "int32->int64",
            "data": "synthetic",
            "config": {"workload": args.workload, "children": int(total), "regions": r_total,
                       "strategy": args.strategy, "w": 128, "stages": len(spec["stages"]),
                       "parallelism": f"whole-region partition x{world}", "gather": gather,
                       "dist_backend": backend, "l2": "inputs larger than L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": bytes_alg / (main_avg / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_alg / (main_avg / 1e3) / 1e9 / peak, "traffic": None,
                         "peak_kind": peak_kind, "kernel": "k_pipeline (rank 0)", "kernel_ms": main_avg,
                         "algorithmic_bytes": bytes_alg},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": p.launches() * args.steps,
            "clocks": clk.summary(), "device_error": code, "gather_check": bool(ok),
        }
        print(json.dumps(line), flush=True)
    if gather == "peer":
        dist.barrier()
        ro.close()
    if comm is not None:
        comm.close()
    dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    import paper_2006_07478_b200 as rs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RS_DIST_BACKEND=gloo + one GPU: every rank shares cuda:0 (a functional test
    # of the multi-rank path on a 1-GPU box; numbers from it are not scaling data)
    backend = os.environ.get("RS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(backend)
        return run_multi(args, rs, torch, dist, world, rank, local, backend)
    dev = torch.device("cuda", local)
    spec = workload_spec(args.workload)
    vals, off = make_inputs(spec, seed=0x5EED + 2, device=dev)
    n = int(off[-1].item() - off[0].item())
    R = int(off.numel() - 1)
    flags = rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING
    p = rs.Pipeline(spec["stages"], spec["agg"], strategy=args.strategy, flags=flags)
    out = p.alloc_outputs(R, dev)
    ws = p.alloc_workspace(R, vals.numel(), dev)

    # ---- device-timed region: W warm-ups, then K steps, synchronised on both sides
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    main_ms = []
    with Clocks(local) as clk:
        clk.wait_ready()                 # sampler running before the warm-up
        for _ in range(args.warmup):
            p.run(vals, off, out, ws)
        torch.cuda.synchronize()
        w0 = time.time()
        t0.record(stream)
        for _ in range(args.steps):
            p.run(vals, off, out, ws)
        t1.record(stream)
        torch.cuda.synchronize()
        clk.mark(w0, time.time())
        time.sleep(0.3)
    total_ms = t0.elapsed_time(t1)
    # per-launch main-kernel time, measured live with events on the launching stream
    for _ in range(max(3, min(args.steps, 10))):
        p.run(vals, off, out, ws)
        main_ms.append(p.kernel_times()[1])
    code = p.check()
    st = p.stats()
    ms_step = total_ms / args.steps
    value = n / (ms_step / 1e3)
    main_avg = statistics.mean(main_ms)
    bytes_alg = alg_bytes(n, R, spec["agg"])
    peak, peak_kind = hbm_peak()
    achieved = bytes_alg / (main_avg / 1e3) / 1e9

    # ---- end-to-end through the C ABI with host buffers (pinned), every step
    e2e = None
    if not args.no_e2e:
        vh = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True)
        vh.copy_(vals)
        oh = torch.empty(off.shape, dtype=off.dtype, pin_memory=True)
        oh.copy_(off)
        outh = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) if o is not None else None for o in out]
        p.run_host(vh, oh, outh[0], outh[1])   # warm-up (device buffers allocated here)
        k = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            p.run_host(vh, oh, outh[0], outh[1])
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / k
        e2e = {"value": n / (e2e_ms / 1e3), "unit": "items/s",
               "h2d_bytes_per_step": int(vals.numel() * vals.element_size() + off.numel() * 8),
               "d2h_bytes_per_step": int(sum(o.numel() * o.element_size() for o in out if o is not None)),
               "ms_per_step": e2e_ms,
               "matches_device_run": all(torch.equal(h, o.cpu()) for h, o in zip(outh, out) if o is not None)}
        del vh, oh, outh

    # ---- parity of the timed run: every region against the oracle's plain fold
    # (outside the timed region; host cores, sharded by whole regions)
    parity = occ_bound = None
    cpu = None
    if not args.no_check or not args.no_cpu:
        import oracle
        vh = vals.cpu().numpy()
        if spec["dtype"] == "u32":
            vh = vh.view(np.uint32)
        elif spec["dtype"] == "u8":
            vh = vh.view(np.uint8)
        oh = off.cpu().numpy()
        if not args.no_check:
            tc = time.perf_counter()
            ref = oracle.brute_sharded(vh, oh, spec["stages"], spec["agg"])
            tc = time.perf_counter() - tc
            mism = 0
            for o, r in zip(out, ref):
                if r is None:
                    continue
                g = o.cpu().numpy()
                g = g.view(r.dtype) if g.dtype.itemsize == r.dtype.itemsize else g.astype(r.dtype)
                mism += int(np.count_nonzero(g != r))
            parity = {"regions": R, "mismatches": mism, "oracle": "plain per-region fold (oracle.brute_sharded)",
                      "threads": len(os.sched_getaffinity(0)), "oracle_s": tc}
            kc = oracle.node_counts(vh, oh, spec["stages"])
            occ_bound = [float(x) for x in oracle.occupancy_bound(kc, 128)]
        if not args.no_cpu:
            cpu = cpu_baseline(vh, oh, spec)

    sweep = configs = None
    if args.sweep:
        del vals, off, out, ws
        torch.cuda.empty_cache()
        sweep = run_sweep(rs, torch, dev, args)
        configs = run_configs(rs, torch, dev, args) + run_taxi(rs, torch, dev, args)

    occ = lane_stats(st)
    if occ_bound is not None:
        for j, o in enumerate(occ):
            o["bound"] = occ_bound[j] if j < len(occ_bound) else None
    if len(spec["stages"]) >= 1:
        occ[-1]["note"] = ("aggregate fused into the last stage (default): its firings are that stage's, its "
                           "items the survivors; see sweep entries with unfused=true for the separate node")
    line = {
        "metric": METRIC, "value": value, "unit": "items/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32->int64", "data": "synthetic",
        "config": {"workload": args.workload, "children": n, "regions": R,
                   "strategy": args.strategy, "w": 128, "stages": len(spec["stages"]),
                   "l2": "inputs (2 GiB) larger than L2; no flush", "parallelism": "regions x1"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_for(args.workload, args.strategy),
                     "peak_kind": peak_kind, "kernel": "k_pipeline", "kernel_ms": main_avg,
                     "algorithmic_bytes": bytes_alg},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": p.launches() * args.steps,
        "clocks": clk.summary(),
        "occupancy": occ,
        "parity": parity,
        "device_error": code,
    }
    if sweep is not None:
        line["sweep"] = sweep
    if configs is not None:
        line["configs"] = configs
    print(json.dumps(line), flush=True)


def run_taxi(rs, torch, dev, args, reps=2):
    """The taxi-style two-stage app: lines of text
    with "{x,y}" pairs; stage 1 keeps the '{' bytes, stage 2 parses, verifies,
    swaps and emits (line, y, x).  Like the paper's replicated DIBS file
    (P:698-705), a 2000-line synthetic corpus is replicated to ~2^28 bytes.
    Signal, tagged and the paper's mix (signal stage 1, tags in stage 2:
    hybrid tag_from=1), each with stage 2 as its own node (unfused)."""
    import synth
    b, off, exp = synth.taxi(2000, seed=5)
    rep = max(1, (1 << 28) // b.size)
    bt = torch.from_numpy(b).to(dev).repeat(rep)
    o1 = torch.from_numpy(off).to(dev)
    offs = torch.cat([o1[:-1] + k * b.size for k in range(rep)] + [torch.tensor([rep * b.size], device=dev)])
    R = offs.numel() - 1
    n = int(bt.numel())
    cap = exp.shape[0] * rep + 64
    res = []
    for strat, kw in (("signal", {}), ("tagged", {}), ("hybrid", {"tag_from": 1})):
        p = rs.Pipeline(synth.taxi_stages(), "emit_pair", strategy=strat,
                        flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | rs.RS_FLAG_UNFUSED, **kw)
        v = torch.empty(2 * cap, dtype=torch.int32, device=dev)
        rg = torch.empty(cap, dtype=torch.int32, device=dev)
        cnt = torch.empty(1, dtype=torch.int64, device=dev)
        ws = p.alloc_workspace(R, n, dev)
        p.run_emit(bt, offs, v, rg, cnt, ws)
        torch.cuda.synchronize()
        ms = []
        for _ in range(reps):
            p.run_emit(bt, offs, v, rg, cnt, ws)
            ms.append(sum(p.kernel_times()))
        t = statistics.median(ms)
        occ = lane_stats(p.stats())
        res.append({"workload": "taxi", "strategy": strat + ("(tag_from=1)" if kw else ""), "children": n,
                    "regions": R, "pairs": int(cnt.item()), "pairs_expected": int(exp.shape[0] * rep),
                    "ms": t, "items_per_s": n / (t / 1e3),
                    "full_rate": [x["full_rate"] for x in occ], "lane_fraction": [x["lane_fraction"] for x in occ],
                    "error": p.check()})
        del p, v, rg, ws
    return res


def run_configs(rs, torch, dev, args):
    """The other BASELINE configs on one GPU: R-MAT graph (D3), text lines (D4),
    Zipf regions (D5, the 8-GPU config's 1-GPU point)."""
    res = []
    for name in ("graph", "text", "zipf"):
        spec = workload_spec(name)
        vals, off = make_inputs(spec, seed=0x5EED + 3, device=dev)
        n, R = int(off[-1].item() - off[0].item()), off.numel() - 1
        for strat in ("signal", "tagged") + (("context",) if spec["dtype"] != "u8" else ()):
            p = rs.Pipeline(spec["stages"], spec["agg"], strategy=strat, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
            out = p.alloc_outputs(R, dev)
            ws = p.alloc_workspace(R, vals.numel(), dev)
            p.run(vals, off, out, ws)
            torch.cuda.synchronize()
            ms = []
            for _ in range(args.sweep_reps):
                p.run(vals, off, out, ws)
                ms.append(sum(p.kernel_times()))
            t = statistics.median(ms)
            st = p.stats()
            res.append({"workload": name, "strategy": strat, "children": n, "regions": R, "ms": t,
                        "items_per_s": n / (t / 1e3),
                        "hbm_frac": alg_bytes(n, R, spec["agg"]) / (t / 1e3) / 1e9 / hbm_peak()[0],
                        "lane_fraction": [x["lane_fraction"] for x in lane_stats(st)], "error": p.check()})
            del out, ws, p
        del vals, off
        torch.cuda.empty_cache()
    return res


def _time_point(rs, torch, dev, args, vals, off, stages, agg, strat, flags=0, bound_kc=None):
    n = int(off[-1].item() - off[0].item())
    R = off.numel() - 1
    p = rs.Pipeline(stages, agg, strategy=strat, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | flags)
    out = p.alloc_outputs(R, dev)
    ws = p.alloc_workspace(R, vals.numel(), dev)
    p.run(vals, off, out, ws)
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.sweep_reps):
        p.run(vals, off, out, ws)
        ms.append(sum(p.kernel_times()))
    st = p.stats()
    t = statistics.median(ms)
    occ = lane_stats(st)
    return {"strategy": strat, "children": n, "regions": R, "ms": t, "items_per_s": n / (t / 1e3),
            "hbm_frac": alg_bytes(n, R, agg) / (t / 1e3) / 1e9 / hbm_peak()[0],
            "lane_fraction": [x["lane_fraction"] for x in occ], "full_rate": [x["full_rate"] for x in occ],
            "error": p.check()}


def run_sweep(rs, torch, dev, args):
    """Items/s and per-node lane fraction vs region length, signal vs tagged
    (BASELINE metric; Figs. 5-6 shape), plus the per-lane context strategy
    (SURVEY §8 f2).  N = 2^29 children per point.  Also: the sawtooth around
    multiples of w, the occupancy bound sum k / (w sum ceil(k/w))
    per node beside each lane fraction (from the oracle's node counts of a
    2^22-child prefix), the unfused aggregate node, and the fp32 variant
    (Fig. 5 push(3.14*v), SUM_F32)."""
    import oracle
    import synth
    res = []
    Ls = [int(x) for x in args.sweep_L.split(",")]
    saw = [int(x) for x in args.sawtooth_L.split(",")] if args.sawtooth_L else []
    N = 1 << 29
    vals = synth.torch_values(N, "i32", seed=11, device=dev)
    stages3 = synth.sweep_stages(3)
    vh_prefix = vals[: 1 << 22].cpu().numpy()
    for dist_ in ("fixed", "var"):
        for L in Ls + saw:
            if dist_ == "fixed":
                lens = torch.full((N // L,), L, dtype=torch.int64, device=dev)
            else:
                lens = synth.torch_lengths(N // L, "var", L=L, seed=L, device=dev)
                cs = torch.cumsum(lens, 0)                # keep the children count <= N
                lens = lens[: int(torch.searchsorted(cs, N, right=True).item())]
            off = synth.torch_offsets(lens)
            oh = off.cpu().numpy()
            rp = max(1, int(np.searchsorted(oh, 1 << 22, side="right")) - 1)   # regions inside the prefix
            bound = [float(x) for x in oracle.occupancy_bound(oracle.node_counts(vh_prefix, oh[:rp + 1], stages3), 128)]
            strats = ("signal", "tagged", "context") if L in Ls else ("signal", "tagged")
            for strat in strats:
                e = _time_point(rs, torch, dev, args, vals, off, stages3, "sum_i64", strat)
                e.update({"dist": dist_, "L": L, "sawtooth": L not in Ls})
                if strat == "signal":
                    e["bound"] = bound
                    # the prepass's rule (rs.h RS_FLAG_SHORT_ON): short-region kernel below 96 children per
                    # region, or below 176 when the regions are of equal length
                    mean = e["children"] / e["regions"]
                    e["kernel"] = "short-region" if mean < 96 or (dist_ == "fixed" and mean < 176) else "general"
                res.append(e)
            if L in Ls and L < 96:             # the general signal kernel at the same point
                e = _time_point(rs, torch, dev, args, vals, off, stages3, "sum_i64", "signal", rs.RS_FLAG_SHORT_OFF)
                e.update({"dist": dist_, "L": L, "sawtooth": False, "kernel": "general", "bound": bound})
                res.append(e)
            if L in (256, 4096):
                e = _time_point(rs, torch, dev, args, vals, off, stages3, "sum_i64", "signal", rs.RS_FLAG_UNFUSED)
                e.update({"dist": dist_, "L": L, "unfused": True, "bound": bound})
                res.append(e)
            del off, lens
    del vals
    torch.cuda.empty_cache()
    # fp32 variant: U[0,1) values, 3 filters on the bit pattern, v' = 3.14f * v, SUM_F32
    fv = synth.torch_values(N, "f32", seed=12, device=dev)
    st4 = synth.sweep_stages(3) + [("scale_f32", 3.14)]
    for L in (256, 4096):
        off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device=dev))
        for strat in ("signal", "tagged"):
            e = _time_point(rs, torch, dev, args, fv, off, st4, "sum_f32", strat)
            e.update({"dist": "fixed", "L": L, "dtype": "f32"})
            res.append(e)
        del off
    del fv
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sweep_fixed_L4096")
    ap.add_argument("--strategy", default=None, choices=["signal", "tagged", "context", "auto"],
                    help="default: signal for the sweep workloads (the headline), auto for zipf / graph / text")
    ap.add_argument("--no-sweep", dest="sweep", action="store_false")
    ap.add_argument("--sweep-L", default="1,4,32,256,4096")
    ap.add_argument("--sweep-reps", type=int, default=2)
    ap.add_argument("--sawtooth-L", default="127,128,129,255,257,4095,4097")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the all-region oracle parity leg")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"])
    args = ap.parse_args()
    if args.strategy is None:
        args.strategy = "signal" if args.workload.startswith("sweep") else "auto"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
