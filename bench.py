#!/usr/bin/env python
"""bench.py — per-channel INT8 KV-key quantization on B200 (arxiv 2601.04719).

One "step" = one pass of the whole hot path over
the workload, through the C ABI on the device-resident inputs:
    kvq_compute_scales (a1 column abs-max, a7 all-reduce MAX when N > 1, a2 /127)
    kvq_quantize       (a3)
    kvq_dequantize     (a4)
    kvq_error_metrics_async (a5 L2 / max-abs, a6 attention-score error, nq = 64)
Workload: BASELINE.json configs[3] (C4: 131072 x 8192 fp32 keys = 1.07e9
elements, 4.3 GB > the 126 MB L2, so no flush is needed), token-sharded over
N ranks (strong scaling).  Rank 0 prints one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1..C4] [--impl kvq|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
`--gpus N` (N > 1) without torchrun re-launches itself under torch.distributed.run with N processes
(one per GPU) and exits non-zero when fewer than N GPUs are visible.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json configs
    "C1": dict(T=1024, D=128, nq=64, desc="keys 1024x128 fp32 (131K elements)"),
    "C2": dict(T=8192, D=1024, nq=64, desc="keys 8192x1024 fp32 (8.4M elements), 64 queries"),
    "C3": dict(T=32768, D=8192, nq=64, desc="keys 32768x8192 fp32 (268M elements)"),
    "C4": dict(T=131072, D=8192, nq=64, desc="keys 131072x8192 fp32 (1.07B elements, 4.3 GB), token-sharded"),
}
METRIC = "quantize+dequantize elements/s and achieved HBM GB/s vs B200 peak at 1/2/4/8 GPUs"
# Algorithmic bytes per element of each pass: what the method itself must move.
SPIN_CYCLES = 100_000  # ~50 us device spin queued ahead of each timed step (keeps launch latency out)
BYTES = {"step": 13, "scales": 4, "quantize": 5, "dequantize": 5, "metrics": 8, "roundtrip": 9, "quantize_dequantize_e4m3": 9,
         "quantize_dequantize_int4": 8.5, "quantize_dequantize_int2": 8.25}


def measured_traffic(kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of `kernel`
    from the committed `ncu --set full` capture summary (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    v = j.get("kernels", {}).get(kernel)
    return None if v is None else {"bytes_per_launch": v["bytes"], "source": j.get("source"), "config": v.get("config")}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm_gbs=j["hbm_gbs"], bf16_tflops=j["bf16_tflops"], sm_max_mhz=j.get("sm_max_mhz", 1965),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, sm_max_mhz=1965, source="fallback (B200_PROFILING.md)")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,clocks.mem")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self, t0=None, t1=None):
        """Median SM clock and active throttle reasons over the samples taken
        inside the wall-clock window [t0, t1] (the timed region)."""
        import datetime
        sm, mx, reasons, mem, pw = [], None, set(), [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, cmax = float(f[2]), float(f[3])
            except ValueError:
                continue
            if t0 is not None and not (t0 - 0.05 <= ts <= t1 + 0.05):
                continue
            sm.append(clk)
            mx = cmax
            try:
                pw.append(float(f[4]))
                if len(f) > 10:
                    mem.append(float(f[10]))
            except ValueError:
                pass
            for n, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "mem_mhz": statistics.median(mem) if mem else None,
                "power_w": statistics.median(pw) if pw else None}


# ----------------------------------------------------------------------------- CPU oracle (baseline / reference arm)
ORACLE_PASSES = ("scales", "quantize", "dequantize", "recon_errors", "attention")


def oracle_step(cfg, rows: int):
    """The oracle as it stands on the first `rows` rows of the workload, one pass at a time:
    scales (a1+a2), quantize (a3), dequantize (a4), L2/max-abs (a5), attention error (a6, nq queries).
    Returns ({pass: seconds}, elements).  Generation is excluded."""
    import oracle
    D, nq = cfg["D"], cfg["nq"]
    K = oracle.fill(rows, D, oracle.SEED_K)
    Q = oracle.fill(nq, D, oracle.SEED_Q)
    t = {}
    t0 = time.perf_counter()
    s = oracle.compute_scales(K)
    t1 = time.perf_counter()
    q = oracle.quantize(K, s)
    t2 = time.perf_counter()
    Kh = oracle.dequantize(q, s)
    t3 = time.perf_counter()
    oracle.recon_errors(K, Kh)
    t4 = time.perf_counter()
    oracle.attention_abs_sum(Q, K, Kh)
    t5 = time.perf_counter()
    t = dict(zip(ORACLE_PASSES, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)))
    return t, rows * D


def oracle_step_all_cores(cfg, rows: int, cores: int):
    """SURVEY §8(d)'s optional all-cores CPU line: the same oracle functions (unchanged, single-threaded C) on
    `cores` row blocks of the same sample, one thread each (ctypes releases the GIL), wall clock per pass.  The
    scales are Alg. 1 (compute_scales, as in the one-core line) per block, combined with an exact max: fl32(m/127)
    is monotonic in m, so the max of the blocks' scales is the scale of the global column max.  L2/max and
    attention are not timed here.  Returns ({pass: seconds}, elements)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    D = cfg["D"]
    K = oracle.fill(rows, D, oracle.SEED_K)
    blocks = [b for b in np.array_split(K, cores) if b.shape[0]]
    blocks = [np.ascontiguousarray(b) for b in blocks]
    t = {}
    with ThreadPoolExecutor(max_workers=len(blocks)) as ex:
        t0 = time.perf_counter()
        s = np.maximum.reduce(list(ex.map(oracle.compute_scales, blocks)))
        t1 = time.perf_counter()
        qs = list(ex.map(lambda b: oracle.quantize(b, s), blocks))
        t2 = time.perf_counter()
        list(ex.map(lambda q: oracle.dequantize(q, s), qs))
        t3 = time.perf_counter()
    t = {"scales": t1 - t0, "quantize": t2 - t1, "dequantize": t3 - t2}
    return t, rows * D


def qdq_seconds(t: dict) -> float:
    """The metric's own mix (quantize+dequantize elements/s): scales + quantize + dequantize."""
    return t["scales"] + t["quantize"] + t["dequantize"]


def cpu_report(t: dict, n: int, steps: int = 1) -> dict:
    """Per-pass oracle seconds and elements/s of the metric's mix (value) and of the whole step."""
    full = sum(t.values())
    return {"value": n * steps / qdq_seconds(t), "unit": "elements/s",
            "per_pass_s": {k: v / steps for k, v in t.items()},
            "per_pass_elements_per_s": {k: n * steps / v for k, v in t.items() if v > 0},
            "full_step_elements_per_s": n * steps / full,
            "value_mix": "scales+quantize+dequantize (a1-a4, the metric's quantize+dequantize); "
                         "full_step_elements_per_s adds a5 L2/max and a6 attention (the GPU step's remaining work)"}


def host_info() -> dict:
    """The host the oracle runs on (CPU model, core count, one core used)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cpu": model, "host_cpu_count": os.cpu_count()}


class one_core:
    """Pin the calling process to one core while the single-threaded oracle is timed."""

    def __enter__(self):
        self.saved = None
        if hasattr(os, "sched_getaffinity"):
            try:
                self.saved = os.sched_getaffinity(0)
                os.sched_setaffinity(0, {min(self.saved)})
            except OSError:
                self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved is not None:
            os.sched_setaffinity(0, self.saved)


def oracle_rows_for(cfg, seconds: float) -> int:
    t, n = oracle_step(cfg, 8)
    per_row = sum(t.values()) / 8
    return max(8, min(cfg["T"], int(seconds / per_row)))


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (plain C, single thread) is this tier's reference arm.
    Under torchrun only rank 0 works; the others exit 0 at once."""
    if rank != 0:
        return
    rows = oracle_rows_for(cfg, 0.5 if args.steps * 1 <= 200 else 0.2)
    for _ in range(args.warmup):
        oracle_step(cfg, rows)
    tot = dict.fromkeys(ORACLE_PASSES, 0.0)
    with one_core():
        for _ in range(args.steps):
            t, n = oracle_step(cfg, rows)
            for k in tot:
                tot[k] += t[k]
    rep = cpu_report(tot, rows * cfg["D"], args.steps)
    value = rep["value"]
    ms = 1e3 * qdq_seconds(tot) / args.steps
    sample = (f"first {rows} rows of {cfg['name']} ({rows}x{cfg['D']} elements) per step; value = scales+quantize"
              f"+dequantize, per-pass seconds include L2/max and attention (nq={cfg['nq']})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (splitmix64 lattice uniform [-1,1), SURVEY §8(d))",
            "config": {"workload": f"{cfg['name']}: {cfg['desc']}", "T": cfg["T"], "D": cfg["D"], "nq": cfg["nq"]},
            "cpu_baseline": {**rep, "cores": 1, "kind": "oracle", "sample": sample, **host_info()},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- the GPU arm
def plan_tail(ntiles: int, ngrp: int, nsm: int, split_max_pieces: int = 640) -> dict:
    """The tensor-core pass's tail plan (csrc/attn_tc.cu tc_plan_tail, same cost model), for gpu_launches."""
    G, W0 = nsm, ntiles // nsm
    whole = {"split": False, "grid": min(ntiles, nsm), "whole": 0, "rt": 0, "pieces": 1}
    whole_cost = -(-ntiles // G) * ngrp
    best, bp = float("inf"), whole
    for W in range(W0, max(0, W0 - 1) - 1, -1):
        rt = ntiles - W * G
        if rt <= 0:
            continue
        for P in range(2, ngrp + 1):
            if ngrp % P or rt * P > split_max_pieces:
                continue
            np_ = rt * P
            cost = W * ngrp + (-(-np_ // G)) * (ngrp // P) + 0.9 * np_ / G + 1.5
            if cost < best:
                best, bp = cost, {"split": True, "grid": G, "whole": W, "rt": rt, "pieces": P}
    return bp if bp["split"] and best < 0.97 * whole_cost else whole


def launches_per_step(args, comm, comm_kind, rows, D):
    """libkvq kernels one step launches (NCCL's own kernels and memsets not counted), per csrc/:
    scales = colmax + finalize (one fused column-max/exchange/finalize kernel with a peer communicator);
    roundtrip = prep (Q split + column records) + attn_tc<2> [+ split_combine when the tail is balanced]
    + reduce_partials (which also writes the result when there is no communicator); metrics alone =
    qsplit + attn_tc<0> [+ split_combine] + reduce_partials; a communicator adds metrics_finalize, and the
    peer one also its metric-exchange kernel."""
    import torch
    nsm = min(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count, 160)
    if os.environ.get("KVQ_TC_RT64", "0") == "1":  # opt-in 64-row roundtrip kernel (rt64.cuh): units of 4
        ntiles, ngrp = (rows + 63) // 64, ((((D + 31) // 32 + 1) // 2) + 3) // 4  # stages of 64 columns
    else:  # the 128-row kernel (attn_tc.cu): 4-K-block work units per tile
        ntiles, ngrp = (rows + 127) // 128, ((D + 31) // 32 + 3) // 4
    combine = 1 if plan_tail(ntiles, ngrp, nsm)["split"] else 0  # split tail -> split_combine_kernel
    peer = comm is not None and comm_kind is not None and comm_kind.startswith(("peer", "nvls"))
    scales = 1 if peer else 2
    tail = 0 if comm is None else (2 if peer else 1)
    if args.format == "int8" and args.pipeline == "step" and comm is None and D <= 256 and rows * D <= (1 << 20):
        return 1  # csrc/step_small.cu: the whole step in one cooperative launch
    l2 = getattr(torch.cuda.get_device_properties(torch.cuda.current_device()), "L2_cache_size", 0)
    if (args.format == "int8" and args.pipeline == "step" and comm is None and D % 16 == 0
            and rows * D * 4 <= l2 // 2):
        # the tensor-core pass with a1 + a2 and the Q split fused in front [+ split_combine] + reduce
        return (3 if os.environ.get("KVQ_TC_RT64", "0") == "1" else 2) + combine
    if args.format == "int8" and args.pipeline in ("fused", "step"):
        if os.environ.get("KVQ_TC_RT64", "0") == "1":
            return scales + 3 + combine + tail
        # whole tiles: the pass's last CTA reduces the partials (no reduce_partials launch)
        return scales + 2 + 2 * combine + tail
    metrics = 3 + combine + tail
    if args.format == "int8":
        return scales + 1 + 1 + metrics  # + quantize + dequantize
    return scales + 1 + metrics          # + the format's fused quantize+dequantize


def run_kvq(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2601_04719_b200 import kvq
    from paper_2601_04719_b200.dist import (enable_nvls, make_comm, make_peer, max_over_ranks, max_over_ranks_vec,
                                            shard_rows)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    kvq.kvq_device_check()
    T, D, nq = cfg["T"], cfg["D"], cfg["nq"]
    row0, rows = shard_rows(T, world, rank)
    # Under torchrun (even with one process) the NCCL exchange path is exercised:
    # kvq_compute_scales all-reduces the column maxima, the metrics their partials.
    # The step's collectives (a7: the scale all-reduce MAX; the metric SUM/MAX): "peer" = a communicator
    # over CUDA-IPC peer memory (kvq_comm_from_peer: column max + exchange + finalize in ONE kernel, the
    # metric partials exchanged by one small kernel; no NCCL), "nccl" = NCCL all-reduces between the
    # kernels.  Without torchrun there is nothing to exchange.
    comm, peer, comm_kind = None, None, None
    if dist.is_available() and dist.is_initialized():
        if args.comm in ("peer", "nvls"):
            try:
                peer = make_peer(rank, world, cfg["D"])
                comm = kvq.Comm.from_peer(peer)
                comm_kind = "peer (CUDA-IPC peer memory, libkvq kvq_comm_from_peer; no NCCL)"
                if args.comm == "nvls":
                    if enable_nvls(peer, rank, world):
                        comm_kind = "nvls (a7 max by multimem.ld_reduce in the NVSwitch; metrics over peer memory)"
                    else:
                        comm_kind = f"peer (NVLS unavailable: {getattr(peer, 'nvls_reason', '')[:80]})"
            except Exception as e:  # e.g. no peer access between the GPUs: NCCL instead
                comm_kind = f"nccl (peer setup failed: {str(e)[:80]})"
        if comm is None:
            comm = make_comm(rank, world)
            comm_kind = comm_kind or "nccl (libkvq kvq_comm_t)"

    def compute_scales():
        kvq.kvq_compute_scales(K, scales, comm=comm, stream=stream)
    stream = torch.cuda.current_stream()

    # device-resident inputs (generated on the GPU by the seeded counter RNG; rank r makes its rows)
    K = kvq.kvq_synth_fill(rows, D, row0=row0, seed=42, device=dev)
    Q = kvq.kvq_synth_fill(nq, D, seed=43, device=dev)
    scales = torch.empty(D, dtype=torch.float32, device=dev)
    Kq = torch.empty((rows, D), dtype=torch.int8, device=dev)
    Kh = torch.empty((rows, D), dtype=torch.float32, device=dev)
    ws = torch.empty(kvq.kvq_roundtrip_workspace_size(rows, D, nq), dtype=torch.uint8, device=dev)
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device=dev)

    def step_separate(ev=None):
        """The four separate ABI calls (a1+a2+a7, a3, a4, a5+a6): 22 B/elem."""
        if ev is not None:
            ev[0].record(stream)
        compute_scales()
        if ev is not None:
            ev[1].record(stream)
        kvq.kvq_quantize(K, scales, Kq, stream=stream)
        if ev is not None:
            ev[2].record(stream)
        kvq.kvq_dequantize(Kq, scales, Kh, stream=stream)
        if ev is not None:
            ev[3].record(stream)
        kvq.kvq_error_metrics_async(K, Kh, Q, scales, out_dev=mout, workspace=ws, comm=comm, stream=stream)
        if ev is not None:
            ev[4].record(stream)

    def step_fused(ev=None):
        """kvq_compute_scales (a1+a2+a7) then kvq_roundtrip (a3+a4+a5+a6 in one pass): 13 B/elem."""
        if ev is not None:
            ev[0].record(stream)
        compute_scales()
        if ev is not None:
            ev[1].record(stream)
        kvq.kvq_roundtrip(K, scales, Q, Kq, Kh, out_dev=mout, workspace=ws, comm=comm, stream=stream)
        if ev is not None:
            ev[2].record(stream)

    Kq8 = torch.empty((rows, D), dtype=torch.uint8, device=dev) if args.format == "e4m3" else None

    def step_e4m3(ev=None):
        """FP8 E4M3 variant (NEXT-1): scales (/448), fused quantize+dequantize, fidelity checks."""
        if ev is not None:
            ev[0].record(stream)
        kvq.kvq_compute_scales_fmt(K, kvq.FMT_E4M3, scales, comm=comm, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        kvq.kvq_quantize_e4m3(K, scales, Kq8, Kh, stream=stream)
        if ev is not None:
            ev[2].record(stream)
        kvq.kvq_error_metrics_async(K, Kh, Q, scales, out_dev=mout, workspace=ws, comm=comm, stream=stream)
        if ev is not None:
            ev[3].record(stream)

    bits = {"int4": 4, "int2": 2}.get(args.format)
    Kp = (torch.empty((rows, kvq.kvq_packed_row_bytes(D, bits)), dtype=torch.uint8, device=dev)
          if bits else None)

    def step_lowbit(ev=None):
        """INT4 / INT2 packed variant (NEXT-3): scales (/7 or /1), fused quantize+dequantize, fidelity checks."""
        if ev is not None:
            ev[0].record(stream)
        kvq.kvq_compute_scales_fmt(K, kvq.FMT_INT4 if bits == 4 else kvq.FMT_INT2, scales, comm=comm, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        kvq.kvq_quantize_packed(K, scales, bits, Kp, Kh, stream=stream)
        if ev is not None:
            ev[2].record(stream)
        kvq.kvq_error_metrics_async(K, Kh, Q, scales, out_dev=mout, workspace=ws, comm=comm, stream=stream)
        if ev is not None:
            ev[3].record(stream)

    wstep = None
    if args.pipeline == "step":
        wstep = torch.empty(kvq.kvq_step_workspace_size(rows, D, nq), dtype=torch.uint8, device=dev)

    def step_one(ev=None):
        """kvq_step: the whole path in ONE ABI call (one cooperative launch for small problems)."""
        if ev is not None:
            ev[0].record(stream)
        kvq.kvq_step(K, Q, scales, Kq, Kh, out_dev=mout, workspace=wstep, comm=comm, stream=stream)
        if ev is not None:
            ev[1].record(stream)

    if args.pipeline == "step":
        step, pass_names = step_one, ["step"]
    elif args.format == "e4m3":
        step, pass_names = step_e4m3, ["scales", "quantize_dequantize_e4m3", "metrics"]
    elif bits:
        step, pass_names = step_lowbit, ["scales", f"quantize_dequantize_{args.format}", "metrics"]
    elif args.pipeline == "fused":
        step, pass_names = step_fused, ["scales", "roundtrip"]
    else:
        step, pass_names = step_separate, ["scales", "quantize", "dequantize", "metrics"]

    if args.graph:
        # the whole step captured once into a CUDA graph (PDL edges and the cooperative launch included) and
        # replayed every step: launch overhead amortized for the launch-bound small configs
        main_stream, stream = stream, torch.cuda.Stream(device=dev)  # the step closures read `stream`
        with torch.cuda.stream(stream):
            for _ in range(3):
                step()
            stream.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
        stream = main_stream

        def step(ev=None):  # noqa: F811
            if ev is not None:
                ev[0].record(stream)
            graph.replay()
            if ev is not None:
                ev[1].record(stream)
        pass_names = ["step"]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # Per-step timing: before every step a barrier (N > 1) and a device sync; then a short
    # device-side spin (torch.cuda._sleep) is queued ahead of the step so the host enqueues all of the step's
    # launches while the stream is still busy (launch latency stays outside the events, as in back-to-back
    # steps).  Each rank times its own step with CUDA events on the launching stream; the step time is the
    # max over ranks, per step; ms_per_step is the median of those, min and mean are reported beside it.
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    se = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        wall0 = time.time()
        for i in range(args.steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            torch.cuda._sleep(SPIN_CYCLES)
            se[i][0].record(stream)
            step(evs[i] if args.pass_events else None)
            se[i][1].record(stream)
        torch.cuda.synchronize()
        wall1 = time.time()
    if world > 1:
        dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in se]
    per_step = max_over_ranks_vec(per_step, dev if world > 1 else None)
    ms = statistics.median(per_step)
    # the same steps back to back (no sync between them), for context
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    b0.record(stream)
    for i in range(args.steps):
        step()
    b1.record(stream)
    torch.cuda.synchronize()
    ms_b2b = max_over_ranks(b0.elapsed_time(b1) / args.steps, dev if world > 1 else None)
    metrics = kvq.metrics_from_device(mout)

    # per-pass device time (events on the launching stream), averaged over the timed steps
    passes = {}
    if args.pass_events:
        for j, nme in enumerate(pass_names):
            passes[nme] = statistics.mean(e[j].elapsed_time(e[j + 1]) for e in evs)
    n_local = rows * D
    pk = peaks()
    pass_report = {}
    for nme, t in passes.items():
        gbs = BYTES[nme] * n_local / (t * 1e-3) / 1e9
        pass_report[nme] = {"ms": t, "algo_bytes_per_elem": BYTES[nme], "GBps": gbs, "frac_hbm": gbs / pk["hbm_gbs"]}
    dom = max(passes, key=passes.get) if passes else None

    # ------------------------------------------------------------------ end to end from pinned host memory
    # Through the public host-buffer call: every step copies K (and Q) host->device from pinned
    # memory, runs the whole path and copies the codes, scales and metrics back.  Two caller
    # streams / workspaces alternate so step i's device->host copy overlaps step i+1's
    # host->device copy (kvq_roundtrip_host_async uses separate H2D and D2H copy engines).
    e2e = None
    if not args.no_e2e and args.format == "int8":
        del Kq, Kh, ws
        torch.cuda.empty_cache()
        K_host = K.cpu().pin_memory()
        Q_host = Q.cpu().pin_memory()
        del K
        torch.cuda.empty_cache()
        wsz = kvq.kvq_roundtrip_host_workspace_size(rows, D, nq)
        slots = []
        for _ in range(2):
            slots.append(dict(stream=torch.cuda.Stream(device=dev),
                              ws=torch.empty(wsz, dtype=torch.uint8, device=dev),
                              sc=torch.empty(D, dtype=torch.float32).pin_memory(),
                              kq=torch.empty((rows, D), dtype=torch.int8).pin_memory(),
                              m=torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8).pin_memory()))

        # One communicator per slot stream: a communicator's exchanges must execute in the same order on every
        # rank, which two streams sharing one communicator would not guarantee (NCCL's rule as well).
        extra = []
        if comm is not None:
            if peer is not None:
                p2 = make_peer(rank, world, D)
                extra = [kvq.Comm.from_peer(p2), p2]
            else:
                extra = [make_comm(rank, world)]
        slots[0]["comm"], slots[1]["comm"] = comm, (extra[0] if extra else None)

        def e2e_step(i):
            sl = slots[i % 2]
            kvq.kvq_roundtrip_host_async(K_host, Q_host, sl["sc"], sl["kq"], sl["m"], sl["ws"], comm=sl["comm"],
                                         stream=sl["stream"])

        for i in range(2):  # warm-up (allocations, first-touch of pinned pages)
            e2e_step(i)
        torch.cuda.synchronize()
        e2e_steps = max(2, min(args.steps, args.e2e_steps))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            e2e_step(i)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        e2e_ms = max_over_ranks(wall_ms, dev if world > 1 else None)
        m_last = kvq.metrics_from_host(slots[(e2e_steps - 1) % 2]["m"])
        e2e = {"value": T * D / (e2e_ms * 1e-3), "unit": "elements/s",
               "h2d_bytes_per_step": rows * D * 4 + nq * D * 4,
               "d2h_bytes_per_step": rows * D + D * 4 + kvq.METRICS_BYTES, "ms_per_step": e2e_ms,
               "steps": e2e_steps, "timing": "host wall clock around the pipelined steps (max over ranks)",
               "api": "kvq_roundtrip_host_async x2 streams (pinned host K/Q -> scales, codes, metrics)",
               "attn_mean_abs": m_last["attn_mean_abs"]}
        if extra:
            torch.cuda.synchronize()
            dist.barrier()
            for x in extra:
                x.destroy()

    if comm is not None:
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
    if peer is not None:
        peer.destroy()
    if rank != 0:
        return
    value = T * D / (ms * 1e-3)
    algo_per_elem = sum(BYTES[n] for n in pass_names)
    algo_bytes = algo_per_elem * T * D
    roofline = None
    if dom:
        t = passes[dom]
        ach = BYTES[dom] * n_local / (t * 1e-3) / 1e9
        tr = measured_traffic(dom) if args.config == "C4" and world == 1 else None
        roofline = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / pk["hbm_gbs"], "traffic": None if tr is None else tr["bytes_per_launch"],
                    "traffic_source": None if tr is None else tr["source"], "peak_source": pk["source"],
                    "algo_bytes_per_elem": BYTES[dom], "algo_bytes_per_launch": BYTES[dom] * n_local,
                    "ms_per_launch": t}
    cpu = None
    if world == 1 and not args.no_cpu:
        with one_core():
            rows_cpu = oracle_rows_for(cfg, args.cpu_seconds)
            t_cpu, n_cpu = oracle_step(cfg, rows_cpu)
        cpu = {**cpu_report(t_cpu, n_cpu), "cores": 1, "kind": "oracle",
               "sample": f"first {rows_cpu} rows of {cfg['name']} ({n_cpu} elements), each pass timed alone: "
                         f"scales, quantize, dequantize, L2/max, attention (nq={nq}); plain C single thread "
                         f"pinned to one core, generation excluded",
               "seconds": sum(t_cpu.values()), **host_info()}
        ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        if ncores > 1:
            t_all, n_all = oracle_step_all_cores(cfg, rows_cpu, ncores)
            cpu["all_cores"] = {"value": n_all / qdq_seconds(t_all), "unit": "elements/s", "cores": ncores,
                                "per_pass_s": t_all,
                                "method": "the same oracle functions on row blocks, one thread per core (ctypes "
                                          "releases the GIL); the blocks' Alg. 1 scales combined with an exact "
                                          "max; scales+quantize+dequantize, same sample"}
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "ms_min": min(per_step), "ms_mean": statistics.mean(per_step),
        "ms_back_to_back": ms_b2b,
        "timing": "per step: barrier + device sync, CUDA events on the launching stream, max over ranks; "
                  "ms_per_step = median over steps",
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (splitmix64 lattice uniform [-1,1), SURVEY §8(d))",
        "config": {"workload": f"{cfg['name']}: {cfg['desc']}", "T": T, "D": D, "nq": nq,
                   "step": "kvq_step (a1, a7, a2, a3, a4, a5, a6 in one ABI call)" if args.pipeline == "step" else
                           ("kvq_compute_scales_fmt(E4M3) -> kvq_quantize_e4m3(+K_hat) -> kvq_error_metrics_async"
                            if args.format == "e4m3" else
                            f"kvq_compute_scales_fmt({args.format.upper()}) -> kvq_quantize_packed(bits={bits}, +K_hat)"
                            " -> kvq_error_metrics_async" if bits else
                            ("kvq_compute_scales(a1,a2,+a7 allreduce MAX) -> kvq_roundtrip(a3 quantize, a4 dequantize,"
                             " a5 L2/max, a6 attention error; one HBM pass)") if args.pipeline == "fused" else
                            "kvq_compute_scales -> kvq_quantize -> kvq_dequantize -> kvq_error_metrics_async"),
                   "pipeline": args.pipeline + (" (CUDA graph)" if args.graph else ""), "format": args.format,
                   "l2_flush": "none needed: inputs larger than L2 (K alone is %.2f GB > 126 MB)" % (4 * T * D / 1e9)
                   if 4 * T * D > 2 * 126e6 else "inputs L2-resident (warm)",
                   "parallelism": f"token-shard x{world}", "comm": comm_kind},
        "hbm": {"GBps": algo_bytes / (ms * 1e-3) / 1e9 / world, "algo_bytes_per_elem": algo_per_elem,
                "frac_of_peak_per_gpu": algo_bytes / (ms * 1e-3) / 1e9 / world / pk["hbm_gbs"]},
        "passes": pass_report, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step(args, comm, comm_kind, rows, D) * args.steps,
        "clocks": clk.summary(wall0, wall1),
        "fidelity": {k: metrics[k] for k in ("l2", "max_abs", "attn_mean_abs", "theoretical_max")},
    }
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(n: int, argv: list, device_count=None, run=subprocess.call) -> int:
    """`python bench.py --gpus N` without torchrun: one process per GPU under torch.distributed.run (the
    driver's own launch line), after checking that N GPUs are visible.  Never falls back to fewer GPUs."""
    if device_count is None:
        import torch
        device_count = torch.cuda.device_count()
    if device_count < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {device_count}", file=sys.stderr, flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return run(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="kvq", choices=["kvq", "reference"])
    ap.add_argument("--pipeline", default="fused", choices=["fused", "separate", "step"],
                    help="fused = kvq_compute_scales + kvq_roundtrip (per-pass events); separate = the four "
                         "calls; step = kvq_step (one call; one cooperative launch for small problems)")
    ap.add_argument("--format", default="int8", choices=["int8", "e4m3", "int4", "int2"],
                    help="int8 = the paper's method (headline); e4m3 = the FP8 variant (NEXT-1); "
                         "int4 / int2 = the packed low-bit variants (NEXT-3)")
    ap.add_argument("--comm", default="peer", choices=["peer", "nvls", "nccl"],
                    help="collectives under torchrun: peer = CUDA-IPC peer memory (a7 fused into the column-max "
                         "kernel, metric partials by one exchange kernel; no NCCL), nvls = the same with the a7 max "
                         "read through NVLS multicast when every GPU can map it, nccl = NCCL all-reduces")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-pass-events", dest="pass_events", action="store_false")
    ap.add_argument("--graph", action="store_true",
                    help="capture the step into one CUDA graph and replay it (per-step events around the replay)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "need >= 3 warm-up steps"
    cfg = dict(CONFIGS[args.config], name=args.config)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    launched = "WORLD_SIZE" in os.environ  # torchrun / torch.distributed.run
    if not launched and args.gpus > 1:
        sys.exit(self_launch(args.gpus, sys.argv[1:]))
    if launched and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one process per GPU")
    if launched:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_kvq(args, cfg, rank, world, local_rank)
    finally:
        if launched:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
