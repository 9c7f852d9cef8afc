#!/usr/bin/env python
"""Benchmark of the B200 VecKM_flow normal-flow path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl b200|reference]

A step = one pass of the hot path (accumulate -> pool -> gather+MLP) over the
workload's synthetic slices, inputs resident in HBM, L2 flushed between steps.
Multi-GPU (torchrun, one rank per GPU), timing the max over ranks:
  default / cfg1-cfg3  every rank its own slice (weak scaling, no collective)
  --workload cfg4      BASELINE's 1000 back-to-back slices split over the ranks
                       (strong scaling, no collective)
  --split spatial      one slice resident on GPU 0, split into row strips inside
                       the step (device partition, NCCL strips, flows gathered
                       back; strong scaling)
`--impl reference` times the reference algorithm's CPU restatement
(oracle/veckm_oracle.py, all host threads) on a bounded sample of the same
workload; on N>1 only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "normal flows/sec (device-timed) at 1/2/4/8 B200; encoder HBM GB/s vs peak"
UNIT = "flows/s"

WORKLOADS = {
    # name: (width, height, events per slice, delta, slices per rank per step, description)
    "cfg1": (346, 260, 100_000, 10, 1, "configs[0]: 346x260 DAVIS slice, 100k events, delta 10"),
    "cfg2": (640, 480, 1_000_000, 10, 1, "configs[1]: synthetic 640x480 slice, 1M events, delta 10"),
    "cfg3": (1280, 720, 4_000_000, 20, 1, "configs[2]: 1280x720 slice, 4M events, delta 20"),
    "cfg4": (346, 260, 200_000, 10, 125, "configs[3]: 346x260 slices of 200k events, 125 per rank per step"),
    "cfg5": (1280, 720, 32_000_000, 10, 1, "configs[4]: 1280x720 slice, 32M events, delta 10 (single GPU)"),
}


def algorithmic_bytes(n, P, P_occ):
    """per slice B = 56n + 516(3P + P_occ), split per kernel."""
    k1 = 24 * n + 516 * P
    k2 = 2 * 516 * P
    k3 = 24 * n + 516 * P_occ + 8 * n
    return k1, k2, k3


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def _synth(n, W, H, seed):
    # bench.synth_workload(..., "uniform_noise") semantics (bench.py:187-190, 209-213)
    g = np.random.default_rng(seed)
    t = g.uniform(0.0, 0.032, size=n)
    x = g.integers(0, W, size=n)
    y = g.integers(0, H, size=n)
    o = np.argsort(t, kind="stable")
    return np.stack([t[o], x[o].astype(np.float64), y[o].astype(np.float64)], axis=1)


def cpu_reference(wl, steps, warmup, budget_s=90.0):
    """Time the reference algorithm (oracle port, all host threads) on a bounded
    sample: accumulate over the slice once (capped at 4M events, linear in n);
    per step, pool + MLP over a strided query subset against that grid (the
    reference's own bench_stage protocol, bench.py:233-285);
    flows/s = 1 / (acc/n + (pool+mlp)/n_sub).  The subset size is picked from a
    calibration step so the whole run stays within ~budget_s."""
    from oracle import veckm_oracle as vo
    from paper_2504_19417_b200.weights import generate_bases, init_weights
    W, H, n, d, _, _ = WORKLOADS[wl]
    cores = os.cpu_count() or 1
    n_acc = min(n, 4_000_000)
    X = _synth(n_acc, W, H, seed=0)
    b = generate_bases(64)
    fr = vo.Freqs(b.time_freqs, b.x_freqs, b.y_freqs, 25.0)
    w = init_weights(64, 128, b, seed=0, dtype=np.float32)
    t = X[:, 0] - X[0, 0]
    xi, yi = X[:, 1].astype(np.int64), X[:, 2].astype(np.int64)
    t_a = time.perf_counter()
    g = vo.accumulate(t, xi, yi, W, H, d, d, fr, 0.016)
    acc_s = time.perf_counter() - t_a
    tab = vo.spatial_table(fr, d, d)

    def pool_mlp(nq):
        q = np.linspace(0, n_acc - 1, nq).astype(np.int64)
        t_p = time.perf_counter()
        emb, _ = vo.pool_threaded(g, tab, t[q], xi[q], yi[q], fr, 0.016, "f32", cores)
        vo.mlp(w.w1, w.b1, w.w2, w.b2, vo.to_features(emb))
        return time.perf_counter() - t_p

    n_cal = 256 * cores
    per_q = pool_mlp(n_cal) / n_cal
    per_step = max(0.05, (budget_s - acc_s) / max(1, steps + warmup))
    nsub = int(min(max(1024, per_step / per_q), 40_000 * cores))
    times = []
    for it in range(warmup + steps):
        dt = pool_mlp(nsub)
        if it >= warmup:
            times.append(dt)
    per_flow = acc_s / n_acc + statistics.median(times) / nsub
    value = 1.0 / per_flow
    sample = (f"{wl}: accumulate over {n_acc} events ({acc_s:.2f} s, once{'' if n_acc == n else ', extrapolated'}) "
              f"+ pool+MLP on {nsub} strided queries per step, {cores} threads; per-flow cost extrapolated")
    return value, cores, sample, statistics.median(times)


def fixed_slice_set(args):
    """Config 4 (BASELINE: 1000 back-to-back slices sharded over the GPUs):
    a fixed slice set split over the ranks, i.e. strong scaling."""
    return args.workload == "cfg4" and not args.slices and args.split != "spatial"


def bench_config(args, world):
    """The `config` of both arms' JSON lines (identical by construction, so
    the driver can match the reference arm to this one)."""
    W, H, n, d, slices, desc = WORKLOADS[args.workload]
    if args.slices:
        slices = args.slices
    spatial = args.split == "spatial"
    extra = {}
    if spatial:
        par = f"spatial{world} (row strips + {d}-row event halo, device partition + gather of owned flows)"
    elif fixed_slice_set(args):
        total = int(os.environ.get("VKM_BENCH_CFG4_SLICES", "1000"))
        slices = -(-total // world)
        extra = {"slices_total_per_step": total}
        par = f"dp{world} (the {total} slices split over the ranks, no collective)"
    else:
        par = f"dp{world} (independent slices per rank, no collective)"
    return {"workload": desc, "sensor": f"{W}x{H}", "events_per_slice": n, "delta": d, **extra,
            "slices_per_rank_per_step": 1 if spatial else slices, "embed_dim": 64, "hidden": 128,
            "mlp_mode": args.mlp_mode, "l2": "flushed between steps (512 MiB write, outside step events)",
            "parallelism": par}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    value, cores, sample, step_s = cpu_reference(args.workload, args.steps, args.warmup, budget_s=args.ref_budget)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if (args.split == "spatial" or fixed_slice_set(args)) else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (uniform noise, seeded per rank), random-init weights D=64/hidden=128",
        "config": bench_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample + " (the reference algorithm on the host cores: oracle/veckm_oracle.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2504_19417_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("VKM_BENCH_SHARED_GPU") == "1"   # test mode: all ranks on cuda:0, gloo
    if shared:
        local = 0
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    W, H, n, d, slices, desc = WORKLOADS[args.workload]
    if args.slices:
        slices = args.slices

    bases = pkg.generate_bases(64, 25.0, (0, 1, 2))
    w = pkg.init_weights(64, 128, bases, seed=0, dtype=np.float32)
    spatial = args.split == "spatial"
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    if spatial:
        # One slice resident on GPU 0, split into row strips inside the timed
        # step (sharding.predict_spatial_device): device row histogram,
        # vkm_select_rows partition + δy halo, NCCL send of each strip,
        # per-rank strip kernels, flows back, vkm_scatter_rows into slice
        # order on GPU 0.  Strong scaling: the slice is fixed as N grows.
        from paper_2504_19417_b200 import sharding
        full = _synth(n, W, H, seed=0) if rank == 0 else None
        t_global = float(full[0, 0]) if rank == 0 else 0.0
        if world > 1:
            box = [t_global]
            dist.broadcast_object_list(box, src=0)
            t_global = box[0]
        full_dev = torch.from_numpy(full).to(dev) if rank == 0 else None
        engines = {}

        def make_engine(h):
            if h not in engines:
                engines[h] = pkg.FlowEngine(W, h, d, d, 0.016, bases, w, device=local, mlp_mode=args.mlp_mode)
            return engines[h]

        def step():
            sharding.predict_spatial_device(make_engine, full_dev, t_global, W, H, d, world, rank)

        slices = 1
        step()                                   # builds this rank's strip engine
        torch.cuda.synchronize()
        eng = next(iter(engines.values()))
        H_eff = eng.height
        host = [full] if rank == 0 else []
        p_occ = [int(len(np.unique(full[:, 2].astype(np.int64) * W + full[:, 1].astype(np.int64))))] if rank == 0 \
            else [0]
        t0s = [t_global]
    else:
        # independent slices: --slices per rank, or for config 4 the 1000
        # back-to-back slices of BASELINE split over the ranks (strong scaling)
        from paper_2504_19417_b200.sharding import slice_range
        if args.workload == "cfg4" and not args.slices:
            total = int(os.environ.get("VKM_BENCH_CFG4_SLICES", "1000"))   # tests shrink it
            mine = slice_range(total, rank, world)
        else:
            mine = range(1000 * rank, 1000 * rank + slices)
        host = [_synth(n, W, H, seed=s) for s in mine]
        slices = len(host)
        H_eff = H
        eng = pkg.FlowEngine(W, H, d, d, 0.016, bases, w, device=local, mlp_mode=args.mlp_mode)
        p_occ = [int(len(np.unique(X[:, 2].astype(np.int64) * W + X[:, 1].astype(np.int64)))) for X in host]
        evs = [torch.from_numpy(np.ascontiguousarray(X)).to(dev) for X in host]
        t0s = [float(X[0, 0]) for X in host]
        flows = [torch.empty((len(X), 2), dtype=torch.float32, device=dev) for X in host]
        if slices > 1:
            # independent slices of one rank: one device buffer, batched launch
            # sequences (vkm_predict_batch: up to 64 slices share each kernel)
            ev_all = torch.cat(evs)
            fl_all = torch.empty((ev_all.shape[0], 2), dtype=torch.float32, device=dev)
            offs_all = np.cumsum([0] + [len(X) for X in host])

        def step():
            if slices > 1:
                eng.predict_batch_device(ev_all, offs_all, t0s, flows=fl_all, stream=stream)
                return
            for s in range(slices):
                eng.predict_device(evs[s], t0s[s], flows=flows[s], stream=stream)
    P = W * H_eff

    # per-kernel CUDA events (vkm_last_timings) sit between kernels and break
    # their programmatic-dependent-launch overlap, so they are recorded on
    # separate profiled steps after the timed ones
    eng.set_profiling(False)
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    launches_per_call = eng.last_timings()[1]

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kern = []
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
            launches += launches_per_call if (slices > 1 or spatial) else launches_per_call * slices
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # Per-kernel times: one launch sequence per profiled step.  Batched
    # slices: the first chunk's worth (the slices one launch sequence takes,
    # pixel budget VKM_BATCH_PIXELS, default 4 Mpx, at most 64 slices).
    kslices = 1
    if slices > 1 and not spatial:
        kslices = int(max(1, min(64, slices, int(os.environ.get("VKM_BATCH_PIXELS", 1 << 22)) // P)))
    eng.set_profiling(True)
    for _ in range(max(5, min(20, args.steps))):
        flush.zero_()
        if slices > 1 and not spatial:
            eng.predict_batch_device(ev_all[: int(offs_all[kslices])], offs_all[: kslices + 1], t0s[:kslices],
                                     flows=fl_all, stream=stream)
        else:
            step()
        t = eng.last_timings()[0]
        if len(t) >= 3 and min(t[:3]) > 0:   # -1: no per-kernel events for this call
            kern.append(t)
    eng.set_profiling(False)
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    if spatial:
        flows_total = n * args.steps
    else:   # every rank's slices (config 4: the 1000 slices in total)
        total_slices = slices
        if world > 1:
            cnt = torch.tensor([float(slices)], dtype=torch.float64, device=dev)
            dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
            total_slices = int(cnt.item())
        flows_total = total_slices * n * args.steps
    value = flows_total / (total_ms / 1e3)

    # ---- end to end through the public host-buffer API (pinned buffers) ----
    # K slices per call through vkm_predict_batch_host (FlowEngine.predict_batch_host,
    # the engine of NormalFlowRegressor.predict_slices): every slice's 24 B/event
    # H2D and 8 B/event D2H are inside the timed region, overlapped with the
    # kernels of the neighbouring slices.  The synchronous one-slice call
    # (vkm_predict_host) is reported beside it.
    e2e = None

    def timed(fn, reps):
        for _ in range(2):
            fn()
        if world > 1:
            dist.barrier()
        t_w = time.perf_counter()
        for _ in range(reps):
            fn()
        dt = time.perf_counter() - t_w
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        return dt

    if not args.no_e2e and spatial:
        # the slice from pinned host memory to GPU 0, the strip split over the
        # ranks, the flows back to pinned host memory (wall clock, max over ranks)
        from paper_2504_19417_b200 import sharding
        pin_in = torch.from_numpy(full).pin_memory() if rank == 0 else None
        pin_out = torch.empty((n, 2), dtype=torch.float32).pin_memory() if rank == 0 else None

        def call_spatial():
            src = pin_in.to(dev, non_blocking=True) if rank == 0 else None
            out = sharding.predict_spatial_device(make_engine, src, t_global, W, H, d, world, rank)
            if rank == 0:
                pin_out.copy_(out, non_blocking=True)
            torch.cuda.synchronize()

        reps = max(3, args.steps // 4)
        e2e_s = timed(call_spatial, reps)
        e2e = {"value": n * reps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 8 * n,
               "steps": reps, "api": "sharding.predict_spatial_device from a pinned host slice (H2D to GPU 0, "
                                     "device partition, NCCL strips, owned flows back, D2H)"}
    elif not args.no_e2e:
        n_e2e = len(host[0])
        # slices per call: --e2e-slices, or by default ~32M events per call
        # (the pipeline's fill and drain amortised; 768 MB of pinned input)
        K = args.e2e_slices if args.e2e_slices > 0 else 32_000_000 // max(1, n_e2e)
        K = max(2, min(K, 64_000_000 // max(1, n_e2e)))   # <= 1.5 GB of pinned input
        pin_ev = torch.empty((K * n_e2e, 3), dtype=torch.float64).pin_memory().numpy()
        pin_out = torch.empty((K * n_e2e, 2), dtype=torch.float32).pin_memory().numpy()
        for k in range(K):
            pin_ev[k * n_e2e:(k + 1) * n_e2e] = host[k % len(host)][:n_e2e]
        offs = np.arange(K + 1, dtype=np.int64) * n_e2e
        ts = np.array([t0s[k % len(t0s)] for k in range(K)], dtype=np.float64)

        def call_batch():
            eng.predict_batch_host(pin_ev, offs, ts, flows=pin_out)

        def call_single():
            eng.predict_host(pin_ev[:n_e2e], t0s[0])

        reps = max(3, args.steps // (4 * K))
        per_slice = world * n_e2e
        e2e_s = timed(call_batch, reps)
        single_s = timed(call_single, max(5, args.steps // 4))
        # the C-ABI packs the f64 rows into 8-byte records on the host for
        # calls of >= 8M events (VKM_HOST_PACK forces it on/off): PCIe bytes
        pk = os.environ.get("VKM_HOST_PACK")
        packed = (pk == "1") if pk is not None else K * n_e2e >= (8 << 20)
        e2e = {"value": per_slice * K * reps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": (8 if packed else 24) * n_e2e, "d2h_bytes_per_step": 8 * n_e2e,
               "input_bytes_per_step": 24 * n_e2e, "host_packed": bool(packed),
               "steps": K * reps, "slices_per_call": K,
               "api": "vkm_predict_batch_host (C-ABI, pinned host buffers of (n,3) f64 rows, copy/compute "
                      "overlap" + ("; rows packed to 8-byte records by host threads" if packed else "") + ")",
               "single_slice": {"value": per_slice * max(5, args.steps // 4) / single_s,
                                "api": "vkm_predict_host (synchronous, one slice per call)"}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    hbm_peak, tc_peak, peak_kind = load_peaks()
    clk_mhz = clk.summary().get("sm_mhz")
    k1b = k2b = k3b = 0
    n_prof = 0
    if spatial:   # rank 0's strip (its events incl. the halo) is what the per-kernel times cover
        from paper_2504_19417_b200 import sharding
        rows = np.bincount(full[:, 2].astype(np.int64), minlength=H)
        se = sharding.strip_events(full, sharding.row_strips(rows, world, d)[0])
        prof = [(len(se.events), int(len(np.unique(se.events[:, 2].astype(np.int64) * W
                                                   + se.events[:, 1].astype(np.int64)))))]
    else:         # the slices of one profiled launch sequence
        prof = [(len(host[i]), p_occ[i]) for i in range(kslices)]
    for n_i, po in prof:
        b1, b2, b3 = algorithmic_bytes(n_i, P, po)
        k1b, k2b, k3b, n_prof = k1b + b1, k2b + b2, k3b + b3, n_prof + n_i
    kernels = None
    roofline = None
    if kern:
        avg = np.mean(np.array(kern), axis=0)
        names = ["accumulate", "pool", "gather_mlp"]
        byts = [k1b, k2b, k3b]
        kernels = {}
        for i, nm in enumerate(names):
            gbs = byts[i] / (avg[i] * 1e-3) / 1e9
            kernels[nm] = {"ms": float(avg[i]), "alg_bytes": int(byts[i]), "gbs": gbs, "frac_hbm": gbs / hbm_peak}
        mlp_tflops = 33280.0 * n_prof / (avg[2] * 1e-3) / 1e12
        kernels["gather_mlp"]["mlp_tflops"] = mlp_tflops
        kernels["gather_mlp"]["frac_tensor_bf16"] = mlp_tflops / tc_peak
        dom = int(np.argmax(avg[:3]))
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                traffic = json.load(fh).get(args.workload, {}).get(names[dom])
        except Exception:
            pass
        a = kernels[names[dom]]["gbs"]
        roofline = {"bound": "hbm", "kernel": names[dom], "achieved": a, "peak": hbm_peak, "unit": "GB/s",
                    "frac": a / hbm_peak, "traffic": traffic, "alg_bytes_per_launch": int(byts[dom]),
                    "peak_kind": peak_kind}
        # Compute roofline beside the HBM one: the encoder groups are bound by
        # instruction issue / the FMA pipe (64 complex phases per event, twice)
        # and the MLP by the tensor pipe.  Warp instructions per launch come
        # from the committed ncu capture of the same workload
        # (profiles/ncu_instr.json, tools/gpu_metrics.sh + tools/ncu_roofline.py)
        # over the group's live CUDA-event time, against 148 SMs x 4 schedulers
        # x the SM clock; pipe activity (FMA-heavy, ALU, tensor) is ncu's own
        # per-kernel measurement of that capture (profiles/ncu_pipes.json).
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_instr.json")) as fh:
                ins = json.load(fh).get(args.workload, {})
            pipes = {}
            pp = os.path.join(ROOT, "profiles", "ncu_pipes.json")
            if os.path.exists(pp):
                with open(pp) as fh:
                    pipes = json.load(fh).get(args.workload, {})
            peak_issue = 148 * 4 * (clk_mhz or 1965.0) * 1e6
            comp = {}
            for g in names:
                if g not in ins:
                    continue
                ach = ins[g] / (kernels[g]["ms"] * 1e-3)
                c = {"bound": "tensor" if g == "gather_mlp" else "issue", "warp_instr_per_launch": ins[g],
                     "issue_achieved": ach, "issue_peak": peak_issue, "issue_frac": ach / peak_issue}
                pg = pipes.get(g) or {}
                for k in ("fmaheavy_pct", "alu_pct", "tensor_pipe_pct"):
                    if k in pg:
                        c[k + "_ncu"] = pg[k]
                comp[g] = c
            if "gather_mlp" in comp:   # F16X3 issues three fp16 MMAs per product: tensor work vs the peak
                comp["gather_mlp"]["tensor_tflops_issued"] = 3 * mlp_tflops if args.mlp_mode in ("auto", "f16x3") \
                    else mlp_tflops
                comp["gather_mlp"]["tensor_frac_issued"] = comp["gather_mlp"]["tensor_tflops_issued"] / tc_peak
            roofline["compute"] = comp
        except Exception:
            pass

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _ = cpu_reference(args.workload, 3, 1, budget_s=20.0)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if (spatial or fixed_slice_set(args)) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform noise, seeded per rank), random-init weights D=64/hidden=128",
        "config": bench_config(args, world),
        "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "kernels": kernels,
        "cpu_baseline": cpu, "clocks": clk.summary(),
        "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--mlp-mode", default="auto", choices=["auto", "fp32", "f16x3", "bf16"])
    ap.add_argument("--slices", type=int, default=0)
    ap.add_argument("--split", choices=["slices", "spatial"], default="slices",
                    help="slices: independent slices per rank (weak); spatial: one slice in row strips (strong)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-slices", type=int, default=0,
                    help="slices per vkm_predict_batch_host call in the e2e leg (0: ~32M events per call, the "
                         "pipeline's fill and drain amortised; at cfg2 8 slices measured 1.5-1.7e9, 32 1.97e9)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=90.0,
                    help="--impl reference: seconds of host work the whole run is sized to")
    args = ap.parse_args()
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    if local_world > 1 and "VKM_HOST_THREADS" not in os.environ:
        # one host pool per rank: share the node's cores instead of every rank
        # starting min(16, cores) threads (read when the library creates its pool)
        try:
            cores = len(os.sched_getaffinity(0))
        except AttributeError:
            cores = os.cpu_count() or 1
        os.environ["VKM_HOST_THREADS"] = str(max(2, min(16, cores // local_world)))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
