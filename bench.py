#!/usr/bin/env python3
"""Benchmark of the B200 EmptyHeaded hot path (BASELINE.json metric:
"triangles counted: input edges/sec and achieved HBM GB/s vs peak (1 B200)").

One STEP = one pass of the whole hot path over
one synthetic input: eh_load_edges (canonicalise, radix sort, dedup, degree
rank, orient, CSR, set layouts, work lists) + eh_count_triangles (eh_free
follows, outside the step's events).  Workload: C3 = RMAT scale 22, edge
factor 16, seed 3 (BASELINE.json configs[2], the configuration the ">= 40 %
of HBM roofline" target names).  `--query k4` (default config C4 =
configs[3]) times the 4-clique step instead: eh_load_edges +
eh_count_4cliques, roofline on B_K4 (eh_alg_bytes_k4).  The printed count is
asserted equal to the oracle's stored value (tests/golden/configs_oracle.json)
when one exists for the config.

  value  = input edges / device time of one step (inputs resident in HBM)
  e2e    = the same metric through the public C ABI with HOST (pinned) inputs,
           every step's H2D copy of the edge list (8 n bytes) and 8-byte D2H of
           its count inside the timed region: eh_count_batch over K steps (the
           same workload uploaded K times); the upload of step i+1 runs on a
           copy stream beside the load + count of step i.  `e2e.single_graph`
           is the synchronous one-graph-at-a-time figure (eh_load_edges from
           host memory + count, nothing overlapped).
  roofline (dominant kernel = the triangle count): achieved = B_tri(tau=32)
           (computed exactly at load: eh_stats.alg_bytes_tri)
           / device time of eh_count_triangles; peak = MEASURED_PEAKS.json hbm_gbs
  cpu_baseline = the CPU oracle (oracle/, untuned) on this host, the paper's
           protocol on the count loop (7 runs, drop the fastest
           and slowest, mean; all host threads) plus its ingest timed once
           (single-threaded qsort; reported separately, as the paper excludes
           loading and index creation from query times)

`--impl reference` times the oracle alone as the reference arm: every step is
one FULL count loop (all host threads) plus the once-timed ingest.
Multi-GPU: the path does not shard (north star "one GPU"):
`--gpus N` under torchrun runs N independent replicas ("replicas only",
DESIGN.md); value = edges processed by all ranks / max-over-ranks time.
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

import synth  # noqa: E402  (input generator; no method arithmetic)


METRIC = "triangles counted: input edges/sec and achieved HBM GB/s vs peak (1 B200)"
METRIC_K4 = "4-cliques counted: input edges/sec and achieved HBM GB/s vs peak (1 B200)"
GOLD = os.path.join(ROOT, "tests", "golden", "configs_oracle.json")


def _workload(cfg, query="tri") -> str:
    q = "4-clique count" if query == "k4" else "triangle count"
    if cfg.kind == "er":
        return f"{cfg.name}: ER G(n={cfg.n}, p={cfg.p}), seed {cfg.seed}; {q}"
    return (f"{cfg.name}: RMAT scale {cfg.scale}, edge factor {cfg.edge_factor}, (a,b,c)=(.57,.19,.19), "
            f"seed {cfg.seed}; {q}")


def _golden(cfg, src, dst, query):
    """The oracle's stored count for this exact input (checksum-matched), else None."""
    if not os.path.exists(GOLD):
        return None
    g = json.load(open(GOLD))["configs"].get(cfg.name)
    if not g or g.get("checksum") != str(synth.checksum(src, dst)):
        return None
    return g.get("four_cliques" if query == "k4" else "triangles")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled every
    10 ms from a thread of this process (the timed region of the default run is a few
    hundred ms, shorter than nvidia-smi's start-up); if NVML is unavailable, an
    `nvidia-smi -lms 100` child started before the warm-up whose lines are kept when they
    arrive inside the [begin(), stop()] window."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.handle = None
        self.samples: list[tuple[float, float, float, int]] = []  # (time, sm, sm_max, reason mask)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.source = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip()]
            phys = int(ids[self.index]) if ids and all(v.strip().isdigit() for v in ids) else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
        return pynvml, h

    def prepare(self):
        """Before the warm-up: open NVML (or start the nvidia-smi child)."""
        try:
            self.nvml, self.handle = self._nvml_handle()
            self.nvml.nvmlDeviceGetClockInfo(self.handle, self.nvml.NVML_CLOCK_SM)
            self.source = "nvml, 10 ms"
            self.t = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.source = "nvidia-smi -lms 100"
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except Exception:
                self.proc = None

    def begin(self):
        """Start of the timed region."""
        if self.nvml is None and self.proc is None and self.source is None:
            self.prepare()
        self.t0 = time.perf_counter()
        if self.nvml is not None:
            self.t.start()

    def _sample_nvml(self):
        n, h = self.nvml, self.handle
        sm = float(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM))
        smax = float(n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM))
        try:
            mask = int(n.nvmlDeviceGetCurrentClocksEventReasons(h))
        except Exception:
            mask = int(n.nvmlDeviceGetCurrentClocksThrottleReasons(h))
        self.samples.append((time.perf_counter(), sm, smax, mask))

    def _poll(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml()
            except Exception:
                break
            self._stop.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            parts = [q.strip() for q in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm, smax = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            mask = 0
            for (_, bit), v in zip(self.REASONS, parts[4:8]):
                if v.lower().startswith("active"):
                    mask |= bit
            self.samples.append((time.perf_counter(), sm, smax, mask))

    def stop(self):
        self.t1 = time.perf_counter()
        self._stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        elif self.proc is not None:
            time.sleep(0.12)  # a line in flight for the end of the window
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml and nvidia-smi unavailable"], "samples": 0}
        tol = 0.0 if self.nvml is not None else 0.1
        win = [q for q in self.samples if self.t0 - tol <= q[0] <= self.t1 + tol]
        mask = 0
        for q in win:
            mask |= q[3]
        return {"sm_mhz": statistics.median(q[1] for q in win) if win else None,
                "sm_max_mhz": max(q[2] for q in win) if win else None,
                "reasons": sorted(nm for nm, bit in self.REASONS if mask & bit), "samples": len(win),
                "source": self.source}


def _dist():
    """(dist, rank, world_size, local_rank).  One process per GPU under torchrun;
    the process group only carries the barrier and the max-over-ranks time
    (replicas only: no data-path collective).  NCCL on GPUs, gloo otherwise."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            backend = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
            dist.init_process_group(backend)
        return dist, dist.get_rank(), ws, int(os.environ.get("LOCAL_RANK", "0"))
    return None, 0, 1, 0


def _max_over_ranks(dist, val: float, device) -> float:
    if dist is None:
        return val
    import torch
    t = torch.tensor([val], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(dist, ws: int, n_in_per_rank: int, local_ms: float, device="cpu"):
    """Whole-job throughput of `ws` independent replicas: every rank processed
    n_in_per_rank input edges in local_ms; the job took the slowest rank's time.
    Returns (value in input edges/s, max ms)."""
    mx = _max_over_ranks(dist, local_ms, device)
    return ws * n_in_per_rank / (mx / 1e3), mx


def _traffic(cfg_name: str, k4: bool):
    """DRAM bytes (read + write) per launch of the count kernels, from the
    committed `ncu --set full` capture (profiles/traffic.json) of this config and
    query, else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(f"{'k4' if k4 else 'tri'}_{cfg_name}_bytes_per_launch")
    return None


def _flush_l2(buf):
    if os.environ.get("BENCH_NOFLUSH") != "1":
        buf.add_(1)  # 512 MiB write: > 2x the 126 MB L2


# ------------------------------------------------------------------ CPU oracle --
def _oracle_protocol(src, dst, query: str, runs: int):
    """The CPU oracle on this host: ingest timed once (it is single-threaded), then
    the full count loop `runs` times with all host threads; the paper's protocol
     keeps the mean of the runs without the fastest and slowest.
    Returns (t_ingest_s, count_mean_s, per-run seconds, threads, count)."""
    import oracle
    threads = oracle.default_threads()
    t0 = time.perf_counter()
    g = oracle.Graph(src, dst)
    t_ing = time.perf_counter() - t0
    times, counts = [], set()
    for _ in range(runs):
        t0 = time.perf_counter()
        counts.add(g.count_4cliques(threads) if query == "k4" else g.count_triangles(threads))
        times.append(time.perf_counter() - t0)
    g.close()
    kept = sorted(times)[1:-1] if len(times) >= 3 else times
    return t_ing, statistics.mean(kept), times, threads, counts.pop() if len(counts) == 1 else sorted(counts)


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg, src, dst, n_in):
    """Reference arm: the CPU oracle as it stands on this host's cores, every timed step
    really executed, sized so that the whole run ends within a few minutes (budget
    BENCH_REF_BUDGET_S, default 300 s of oracle time):

      "ingest + count"  each step = oracle ingest + the full count loop (the GPU arm's step)
                        when (warmup + steps) of them fit the budget;
      "count loop"      else each step = one FULL count loop; the oracle's (single-threaded)
                        ingest runs once, before the timed region, and is reported separately
                        (the paper's protocol excludes loading and index creation);
                        value = n_in / count-loop time, which flatters the oracle;
      "slice"           else each step counts one 1/S slice of the outer x loop (another slice
                        each step) and value = (n_in / S) / slice time.

    ms_per_step is the measured wall time of one step in every mode (steps x ms_per_step is
    inside the run's wall clock)."""
    import oracle
    dist, rank, ws, _ = _dist()
    if rank != 0:
        return
    threads = oracle.default_threads()
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "300"))
    k4 = args.query == "k4"
    count = (lambda g: g.count_4cliques(threads)) if k4 else (lambda g: g.count_triangles(threads))
    t0 = time.perf_counter()
    g = oracle.Graph(src, dst)
    t_ing = time.perf_counter() - t0
    m_und, n_act = int(g.m), int(g.n_vertices)
    t0 = time.perf_counter()
    probe_count = count(g)  # the first warm-up step's count loop; sizes the mode
    t_probe = time.perf_counter() - t0
    total = args.warmup + args.steps
    counts = {probe_count}
    times = []
    if total * (t_ing + t_probe) <= budget:
        mode, S = "ingest + count", 1
        g.close()
        for i in range(total):
            t0 = time.perf_counter()
            g = oracle.Graph(src, dst)
            counts.add(count(g))
            dt = time.perf_counter() - t0
            g.close()
            if i >= args.warmup:
                times.append(dt)
        edges_per_step = n_in
    elif total * t_probe <= budget:
        mode, S = "count loop", 1
        for i in range(1, total):  # the probe was warm-up step 0 (or, with --warmup 0, an extra one)
            t0 = time.perf_counter()
            counts.add(count(g))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        if len(times) < args.steps:  # --warmup 0: the probe does not count as a timed step
            t0 = time.perf_counter()
            counts.add(count(g))
            times.append(time.perf_counter() - t0)
        g.close()
        edges_per_step = n_in
    else:
        S = int(-(-total * t_probe // budget))
        mode = "slice"
        nv = g.n_vertices
        rng_count = g.count_4cliques_range if k4 else g.count_triangles_range
        counts = set()
        for i in range(total):
            x0, x1 = nv * (i % S) // S, nv * (i % S + 1) // S
            t0 = time.perf_counter()
            rng_count(x0, x1, threads)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        g.close()
        counts = {probe_count}
        edges_per_step = n_in / S
    step = statistics.mean(times)
    value = edges_per_step / step
    what = "4-clique" if k4 else "triangle"
    sample = {"ingest + count": f"every step = the oracle ingest of the full {cfg.name} input (single-threaded) + the full "
                                f"{what} count loop ({threads} threads)",
              "count loop": f"every step = one full {cfg.name} {what} count loop ({threads} threads, mean {step:.2f} s); the "
                            f"oracle ingest of the full input ran once before the timed region ({t_ing:.2f} s, "
                            f"single-threaded) and is NOT in the step (PAPER.md:756 excludes loading and index creation)",
              "slice": f"every step = the {what} count over one 1/{S} slice of the outer x loop of {cfg.name} (another "
                       f"slice each step, {threads} threads); value = (n_in / {S}) / slice time; full loop {t_probe:.1f} s, "
                       f"ingest {t_ing:.1f} s"}[mode] + f"; host: {_cpu_model()}"
    line = {"impl": "reference", "metric": METRIC_K4 if k4 else METRIC, "value": value,
            "unit": "input edges/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": _workload(cfg, args.query), "n_input": n_in, "m_undirected": m_und, "n_active": n_act,
                       "parallelism": f"{threads} host threads", "reference_step": mode},
            "count": counts.pop() if len(counts) == 1 else sorted(counts),
            "cpu_baseline": {"value": value, "unit": "input edges/s", "cores": threads, "kind": "oracle",
                             "sample": sample, "ingest_s": t_ing, "ingest_threads": 1,
                             "count_s": times if mode != "ingest + count" else None, "full_count_loop_s": t_probe},
            "e2e": {"value": value, "unit": "input edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm --
def run_gpu(args, cfg, src, dst, n_in):
    import torch
    import paper_1503_02368_b200 as eh

    dist, rank, ws, local = _dist()
    k4 = args.query == "k4"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    peak, peak_kind = _peaks()

    # inputs resident in HBM before the timed region (value); pinned host copies (e2e)
    d_src = torch.from_numpy(src.view(np.int32)).to(dev)
    d_dst = torch.from_numpy(dst.view(np.int32)).to(dev)
    h_src = torch.from_numpy(src.view(np.int32)).pin_memory()
    h_dst = torch.from_numpy(dst.view(np.int32)).pin_memory()
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)  # 512 MiB
    torch.cuda.synchronize()

    def one_step(host: bool, want_stats: bool = False):
        """Returns (t_step_ms, t_count_ms, count, stats or None).  Statistics are
        computed on demand by the library, outside the step's events."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            if host:
                g = eh.Graph(h_src, h_dst, stream=stream)
            else:
                g = eh.Graph(d_src, d_dst, stream=stream)
            ev[1].record(stream)
            c = g.count_4cliques() if k4 else g.count_triangles()
            ev[2].record(stream)
            stream.synchronize()
            st = None
            if want_stats:
                st = g.stats()
                if k4:
                    st.alg_bytes_k4 = g.alg_bytes_k4()
            g.close()
        stream.synchronize()
        return ev[0].elapsed_time(ev[2]), ev[1].elapsed_time(ev[2]), c, st

    clocks = ClockSampler(local)
    clocks.prepare()
    # warm-up
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            _flush_l2(flush)
        one_step(False)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.begin()
    l0 = eh.launch_count()
    step_ms, count_ms, counts = [], [], set()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            _flush_l2(flush)  # outside the per-step events
        t, tc, c, _ = one_step(False)
        step_ms.append(t)
        count_ms.append(tc)
        counts.add(c)
    launches = (eh.launch_count() - l0) / max(1, args.steps)
    st = one_step(False, want_stats=True)[3]  # untimed: B_tri and sizes for the report
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    # e2e (single graph) through the C ABI with host buffers (H2D inside the timed
    # region); one untimed host-path step first (the pool grows for the upload buffer)
    one_step(True)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        with torch.cuda.stream(stream):
            _flush_l2(flush)
        t, _, c, _ = one_step(True)
        e2e_ms.append(t)
        counts.add(c)
    # e2e (pipelined): eh_count_batch over K host copies of the workload (each step
    # uploads its 8 n bytes again; inputs > L2, so no flush between the steps)
    # (library streams of their own, blocking w.r.t. the legacy default stream, so
    # events recorded there bracket the whole batch on the device)
    K = max(4, args.steps)
    lists = [(h_src, h_dst)] * K
    q = "4cliques" if k4 else "triangles"
    eh.count_batch(lists[:4], q)  # untimed warm-up (pools, streams)
    legacy = torch.cuda.default_stream(dev)
    with torch.cuda.stream(legacy):
        _flush_l2(flush)
    eb = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    eb[0].record(legacy)
    bc = eh.count_batch(lists, q)
    eb[1].record(legacy)
    torch.cuda.synchronize()
    counts.update(bc)
    batch_ms = eb[0].elapsed_time(eb[1]) / K
    if len(counts) != 1:
        raise RuntimeError(f"non-deterministic counts: {counts}")
    T = counts.pop()
    gold = _golden(cfg, src, dst, args.query)
    if gold is not None and T != gold:
        raise RuntimeError(f"count {T} differs from the oracle's stored value {gold}")
    mean_step = statistics.mean(step_ms)
    mean_count = statistics.mean(count_ms)
    mean_e2e = statistics.mean(e2e_ms)
    value, mean_step_max = aggregate(dist, ws, n_in, mean_step, dev)
    e2e_single, mean_e2e_max = aggregate(dist, ws, n_in, mean_e2e, dev)
    e2e_value, batch_ms_max = aggregate(dist, ws, n_in, batch_ms, dev)
    if rank != 0:
        return
    alg = st.alg_bytes_k4 if k4 else st.alg_bytes_tri
    achieved = alg / (mean_count / 1e3) / 1e9
    line = {
        "metric": METRIC_K4 if k4 else METRIC,
        "value": value, "unit": "input edges/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_step_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": {"workload": _workload(cfg, args.query),
                   "n_input": n_in, "m_undirected": st.m_undirected, "n_active": st.n_active,
                   "parallelism": "replicas only" if ws > 1 else "1 GPU",
                   "l2": "512 MiB flush write between timed steps (outside the per-step events); inputs "
                         f"{8 * n_in / 1e6:.0f} MB",
                   "step": ("eh_load_edges(device inputs) + " + ("eh_count_4cliques" if k4 else "eh_count_triangles")
                            + " (eh_free after the step's events)")},
        ("four_cliques" if k4 else "triangles"): T,
        "oracle_golden_match": gold is not None,
        "count_ms": mean_count, "load_ms": mean_step - mean_count,
        "count_edges_per_s": n_in / (mean_count / 1e3),
        ("four_cliques_per_s" if k4 else "triangles_per_s"): T / (mean_count / 1e3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _traffic(cfg.name, k4), "peak_kind": peak_kind,
                     "kernel": "k_k4_* (eh_count_4cliques)" if k4 else "k_tri_* (eh_count_triangles)",
                     "alg_bytes": "B_K4(tau=32)" if k4 else "B_tri(tau=32)", "alg_bytes_per_launch": alg},
        "e2e": {"value": e2e_value, "unit": "input edges/s",
                "h2d_bytes_per_step": 8 * n_in, "d2h_bytes_per_step": 8, "ms_per_step": batch_ms_max,
                "api": f"eh_count_batch over {K} steps from pinned host memory: the upload of step i+1 runs "
                       "on a copy stream beside the load + count of step i (one lane at this size; two lanes "
                       "of alternate steps for lists of <= 2^23 edges)",
                "single_graph": {"value": e2e_single, "ms_per_step": mean_e2e_max,
                                 "api": "eh_load_edges_ex(host inputs) + count + eh_free, one step at a time"}},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if not args.no_cpu_baseline and ws == 1:
        runs = args.cpu_runs or (3 if k4 else 7)
        t_ing, t_cnt, per_run, threads, oc = _oracle_protocol(src, dst, args.query, runs)
        if oc != T:
            raise RuntimeError(f"GPU count {T} differs from the oracle's {oc}")
        line["cpu_baseline"] = {
            "value": n_in / (t_ing + t_cnt), "unit": "input edges/s", "cores": threads, "kind": "oracle",
            "sample": (f"full {cfg.name} input: oracle ingest timed once ({t_ing:.1f} s, single-threaded qsort) + "
                       f"the full {'4-clique' if k4 else 'triangle'} count loop, {runs} runs on {threads} threads, "
                       f"mean without the fastest and slowest ({t_cnt:.2f} s; PAPER.md:756); host: {_cpu_model()}"),
            "ingest_s": t_ing, "ingest_threads": 1, "count_s": t_cnt, "count_runs_s": per_run,
            "count_value": n_in / t_cnt}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="eh", choices=["eh", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(synth.CONFIGS),
                    help="default C3 (triangles) or C4 (--query k4)")
    ap.add_argument("--query", default="tri", choices=["tri", "k4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-runs", type=int, default=0, help="oracle count-loop runs (default 7; 3 for k4)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "C4" if args.query == "k4" else "C3"
    if args.warmup < 3 and args.impl == "eh":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    cfg = synth.CONFIGS[args.config]
    src, dst = cfg.generate()
    n_in = int(src.size)
    if args.impl == "reference":
        run_reference(args, cfg, src, dst, n_in)
    else:
        run_gpu(args, cfg, src, dst, n_in)


if __name__ == "__main__":
    main()
