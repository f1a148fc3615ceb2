#!/usr/bin/env python
"""Benchmark: rendered receiver-query spectra/s (BASELINE.json metric).

Workload (N=1, BASELINE.json configs[1]): synthetic scene of 100k Gaussians
(l_max=2, C=1), one transmitter, a batch of 1024 unseen receiver positions,
90x360 az/el spectrum + RSSI per receiver, receiver-conditioned (full mode,
F=6 d=64 d_c=16 S=16, 32^3 occupancy).  One step = build the transmitter
state (projection, basis, tile sort, FP64 blend walk) + render the receiver
batch (conditioning fused with the FLE reduction, compositing, spectrum/RSSI
epilogue).  Multi-GPU (torchrun): weak scaling, every rank renders its own
1024-receiver shard of the query grid against the replicated scene; no
data-path collective (timing uses a barrier and a max-reduce only).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rendered Rx-query spectra/sec at N Gaussians (1/2/4/8 B200) vs host-CPU ref"
UNIT = "spectra/s"
TX = (0.3, -0.2, 0.1)
BOX_LO, BOX_HI = (-4.0, -3.0, -1.5), (4.0, 3.0, 1.5)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--gaussians", type=int, default=100_000)
    ap.add_argument("--rx", type=int, default=1024, help="receivers per rank per step")
    ap.add_argument("--n-theta", type=int, default=90)
    ap.add_argument("--n-phi", type=int, default=360)
    ap.add_argument("--cpu-sample", type=int, default=0, help="receivers in the CPU baseline sample (0=auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-batch", type=int, default=16, help="(tx, rx) samples per GPU per training step")
    ap.add_argument("--no-config3", action="store_true", help="skip the coverage-table (config 3) leg")
    ap.add_argument("--no-config5", action="store_true", help="skip the 2M / 180x720 (config 5) leg")
    ap.add_argument("--no-lmax9", action="store_true", help="skip the config-2 l_max = 9 (L = 100) leg")
    ap.add_argument("--no-config1", action="store_true", help="skip the config-1 single-query latency leg")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args):
    return {"workload": "config2: synthetic scene, 1 Tx x receiver batch, spectrum + RSSI",
            "gaussians": args.gaussians, "l_max": 2, "channels": 1,
            "grid": f"{args.n_theta}x{args.n_phi}", "tile": 8,
            "rx_per_rank": args.rx, "conditioning": "full F6 d64 dc16 S16 R32",
            "step": "build_tx_state + render_queries(batch)",
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": "receiver shards, scene replicated"}


def make_inputs(args, lib, rank, world):
    """Replicated scene; this rank's shard of the world * rx receiver query set."""
    from paper_2605_24290_b200.dist import shard_range
    sc = lib.synth_scene(args.gaussians, 2, 1, 7)
    b, e = shard_range(world * args.rx, rank, world)
    rx = lib.synth_points(world * args.rx, 11, "bench.rx", BOX_LO, BOX_HI, 0.05)[b:e]
    return sc, rx


# ---------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.thread = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{device}.csv")

    def start(self):
        # NVML in a thread, ~1 ms period: the timed region is tens of ms, shorter
        # than nvidia-smi's loop period (kept as the fallback)
        self.samples = []
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # the CUDA device by PCI bus id (NVML indices ignore CUDA_VISIBLE_DEVICES)
                import torch
                pr = torch.cuda.get_device_properties(self.device)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.stop_ev = threading.Event()
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}

            def run():
                while not self.stop_ev.is_set():
                    try:
                        mhz = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, [n for n, b in bits.items() if r & b]))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.001)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if getattr(self, "thread", None) is not None:
            self.stop_ev.set()
            self.thread.join(timeout=5)
            if not self.samples:
                return None
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            with open(self.path, "w") as fh:  # the raw samples, for the record
                for mhz, rs in self.samples:
                    fh.write(f"{mhz},{self.max_mhz},{'|'.join(rs)}\n")
            reasons = sorted({n for _, rs in self.samples for n in rs})
            return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(self.samples), "source": "NVML, ~1 ms period"}
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU reference
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_setup(args):
    """The reference model (oracle/_ref: the unmodified reference sources, see
    oracle/Makefile) built once: scene, conditioning, occupancy."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # cpu_baseline leg: the one place bench.py executes oracle/
    chk = O.reference()
    if chk is None:
        raise RuntimeError("oracle/_ref/librxgs_ref.so missing (build() compiles it where /root/reference exists)")
    sc = chk.synth_scene(args.gaussians, 2, 1, 7)
    h = chk.scene(sc, "spectrum")
    lo, hi = chk.scene_bounds(h, 0.0)
    cfg = O.cond_cfg()
    params = chk.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    olo, ohi = chk.scene_bounds(h, 0.1)
    occ = chk.build_occupancy(h, 32, olo, ohi)
    cond = chk.cond(cfg, params, occ, olo, ohi)
    return chk, h, cond, O.Grid(args.n_theta, args.n_phi, 8, 1.0)


def cpu_reference_run(args, sample, threads, setup=None):
    """One bounded sample of the config-2 step on the reference's CPU path:
    build_tx_state + `sample` receivers (conditioning, render, aggregation)."""
    chk, h, cond, grid = setup if setup is not None else cpu_reference_setup(args)
    rx = chk.synth_points(sample, 11, "bench.rx", BOX_LO, BOX_HI, 0.05)
    secs, _, _ = chk.bench_queries(h, cond, grid, TX, rx, threads)
    return secs, "reference"


# ---------------------------------------------------------------- GPU arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if args.gpus != world and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} rank(s)", file=sys.stderr)
    n_dev = torch.cuda.device_count()
    shared = world > n_dev  # functional check only: ranks share GPUs, gloo plumbing
    if shared:
        print(f"bench: {world} ranks on {n_dev} GPU(s): ranks share devices over gloo (NOT a scaling "
              f"measurement)", file=sys.stderr)
        local = local % n_dev
    torch.cuda.set_device(local)
    if world > 1 and not shared:
        # NCCL's communicator lines (rank / nranks / transport) on the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        warm = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(warm)  # communicator up before any timing
        torch.cuda.synchronize()
    elif world > 1:
        dist.init_process_group("gloo")
    from paper_2605_24290_b200 import capi

    dev = torch.device("cuda", local)
    sc, rx_np = make_inputs(args, capi, rank, world)
    ctx = capi.Context(local)
    # One explicit stream for torch (flush, events) and the library: the
    # legacy default stream (handle 0) cannot be shared with the C-ABI.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    scene = ctx.scene(sc, "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg()
    params = capi.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    cond = ctx.cond(cfg, params)
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(args.n_theta, args.n_phi, 8, 1.0)
    tx = np.array(TX)
    n = args.rx
    P = grid.cells

    rx_dev = torch.from_numpy(rx_np).to(dev)
    spec_dev = torch.empty((n, args.n_theta, args.n_phi), dtype=torch.float32, device=dev)
    rssi_dev = torch.empty(n, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_device():
        st = scene.tx_state(tx, grid)
        scene.render_queries(cond, st, rx_dev, spec_dev, rssi_dev)
        return st

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    last = None
    for _ in range(args.warmup):  # same pattern as the timed loop (fills the state pool)
        last = step_device()
    barrier()

    # ---------------- device-resident timed region (no per-kernel events inside it)
    clocks = ClockSampler(local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    barrier()
    last = None
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (outside the events)
        starts[i].record(stream)
        last = step_device()  # the previous step's state is released (buffers recycled)
        ends[i].record(stream)
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    ms_steps = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_local = sum(ms_steps) / len(ms_steps)
    del last
    # ---------------- per-kernel times (CUDA events on the launch stream), a separate pass
    ctx.reset_stats()
    ctx.profile(True)
    for i in range(max(2, min(args.steps, 3))):
        flush.fill_(float(i))
        last = step_device()
    torch.cuda.synchronize(dev)
    cond_ms, cond_n, cond_rows = ctx.kernel_stats("cond_signal")
    comp_ms, comp_n, _ = ctx.kernel_stats("composite")
    walk_ms, _, _ = ctx.kernel_stats("walk")
    ctx.profile(False)
    stats = last.stats()
    del last

    ms = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_max = float(ms.item())
    value = world * n / (ms_max / 1e3)

    # ---------------- end-to-end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        rx_host = torch.from_numpy(rx_np.copy()).pin_memory()
        spec_host = torch.empty((n, args.n_theta, args.n_phi), dtype=torch.float32).pin_memory()
        rssi_host = torch.empty(n, dtype=torch.float32).pin_memory()
        rx_h, spec_h, rssi_h = rx_host.numpy(), spec_host.numpy(), rssi_host.numpy()
        tx_h = np.array(TX)

        def step_e2e():
            st = scene.tx_state(tx_h, grid)
            scene.render_queries(cond, st, rx_h, spec_h, rssi_h)

        for _ in range(max(1, args.warmup)):
            step_e2e()
        barrier()
        t_ms = []
        for i in range(args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize(dev)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            t0 = time.perf_counter()
            step_e2e()
            e.record(stream)
            torch.cuda.synchronize(dev)
            t_ms.append(max((time.perf_counter() - t0) * 1e3, s.elapsed_time(e)))
        em = torch.tensor([sum(t_ms) / len(t_ms)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(em, op=dist.ReduceOp.MAX)
        e2e = {"value": world * n / (float(em.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(n * 3 * 8 + 3 * 8),
               "d2h_bytes_per_step": int(n * P * 4 + n * 4),
               "ms_per_step": float(em.item())}

    # ---------------- roofline of the dominant kernel (cond_signal)
    d, S, L, C = 64, 16, 9, 1
    flop_row = 2 * (6 * d + d * d + 4 * C * d) + S * 30 + 20 + L * C * 16
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 1590.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        pk = json.load(open(peaks_path))
        peak, peak_src = float(pk.get("bf16_tflops", 1590.0)), "measured bf16_tflops (MEASURED_PEAKS.json)"
    roofline = None
    traffic = None
    tpath = next((os.path.join(ROOT, "profiles", f"{t}_traffic.json") for t in ("r2", "r1")
                  if os.path.exists(os.path.join(ROOT, "profiles", f"{t}_traffic.json"))), "")
    ncu_pipes = None
    if os.path.exists(tpath):  # dram bytes of the same kernel from the committed ncu --set full capture
        tj = json.load(open(tpath))
        traffic = tj.get("k_cond_tc", {}).get("dram_bytes_per_launch")
        # ncu pipe evidence of the config-2 kernels (same capture): FP32 / tensor pipe
        # and issue utilisation, achieved DRAM GB/s and its fraction of the measured HBM peak
        hbm = 6548.2
        if os.path.exists(peaks_path):
            hbm = float(json.load(open(peaks_path)).get("hbm_gbs", hbm))
        ncu_pipes = {}
        for kn in ("k_cond_tc", "k_fle_gemm", "k_composite_tc", "k_walk"):
            r = tj.get(kn)
            if not r or r.get("fp32_pipe_pct") is None:
                continue
            ncu_pipes[kn] = {"fp32_pipe_pct": round(r["fp32_pipe_pct"], 1),
                             "tensor_pipe_pct": round(r["tensor_pipe_pct"], 1),
                             "fp64_pipe_pct": round(r["fp64_pipe_pct"], 1),
                             "issue_active_pct": round(r["issue_active_pct"], 1),
                             "dram_gbps": round(r["dram_gbps"], 1),
                             "hbm_frac": round(r["dram_gbps"] / hbm, 3)}
        ncu_pipes = ncu_pipes or None
    if cond_n:
        per_launch_rows = cond_rows / cond_n
        avg_ms = cond_ms / cond_n
        achieved = flop_row * per_launch_rows / (avg_ms / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak,
                    # with tcgen05 at 3 MMAs per product (bf16x3) the pipe's
                    # usable peak for the same algorithmic FLOP is peak / 3
                    "frac_of_bf16x3_peak": achieved / (peak / 3.0), "traffic": traffic, "traffic_unit": f"bytes per launch ({os.path.relpath(tpath, ROOT) if tpath else 'no capture'})",
                    "kernel": "cond_signal = k_fle_gemm (FLE reduction, tcgen05 GEMM) + k_cond_tc (probe + local MLP on tcgen05 + affine)",
                    "pipe": "tcgen05 bf16x3 (layers 1-2, FLE GEMM) + FP32 SIMT on FFMA2 (probe, layer 3, affine)", "peak_source": peak_src,
                    "flop_per_row": flop_row, "rows_per_launch": per_launch_rows,
                    "kernel_ms": avg_ms,
                    "share_of_step": (cond_ms / cond_n) / ms_local,
                    "composite_ms": comp_ms / max(comp_n, 1), "walk_ms": walk_ms / max(comp_n, 1),
                    "ncu_pipes": ncu_pipes,
                    "ncu_pipes_source": f"{os.path.relpath(tpath, ROOT) if tpath else 'no capture'} "
                                        "(ncu --set full, one launch each, cold cache)"}

    train = None if args.no_train else bench_train(args, capi, ctx, scene, cond, grid, stream, dev, rank, world)
    del scene, cond
    cov = None if args.no_config3 else bench_coverage(args, capi, ctx, stream, dev, rank, world)
    large = None if args.no_config5 else bench_large(args, capi, ctx, stream, dev, rank, world)
    lmax9 = None if args.no_lmax9 else bench_lmax9(args, capi, ctx, stream, dev, rank, world)
    c1 = None if args.no_config1 or rank != 0 else bench_config1(args, capi, ctx, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.cpu_sample or 256
        try:
            secs, kind = cpu_reference_run(args, sample, threads)
            cpu = {"value": sample / secs, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                   "sample": f"{sample} receivers of the same workload (K={args.gaussians}, "
                             f"{args.n_theta}x{args.n_phi}), build_tx_state + condition_forward (fanned over "
                             f"{threads} threads) + render_field (chunks of 16, {threads} threads) + "
                             f"spectrum/RSSI aggregation; {secs:.1f} s wall"}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32 (FP64 geometry/walk)", "data": "synthetic",
                "config": workload(args), "e2e": e2e, "gpu_launches": int(launches),
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
                "train_config4": train, "config1": c1, "config2_lmax9": lmax9, "config3": cov,
                "config5": large, "tx_state": stats}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_train(args, capi, ctx, scene, cond, grid, stream, dev, rank, world):
    """BASELINE config 4: Stage-II training step (conditioning + compositing
    forward and backward, spectrum L1) on B samples per GPU, the flat f64
    gradient all-reduced over NCCL when world > 1, then Adam.  Geometry is
    frozen (Stage II), so the transmitter state is cached (trainer.cpp:417-427)."""
    import torch
    import torch.distributed as dist
    from paper_2605_24290_b200.dist import allreduce_grads, max_over_ranks, shard_range

    B = args.train_batch
    b, e = shard_range(world * B, rank, world)
    rx = capi.synth_points(world * B, 23, "bench.train.rx", BOX_LO, BOX_HI, 0.05)[b:e]
    rng = np.random.default_rng(29 + rank)
    targets = torch.from_numpy(rng.uniform(0.0, 2.0, (B, grid.cells)).astype(np.float32)).to(dev)
    rx_d = torch.from_numpy(rx).to(dev)
    st = scene.tx_state(np.array(TX), grid)

    def time_trainer(hyper, geometry=None):
        sc_t, cond_t = scene, cond
        if geometry:  # joint step: own copy of the model, its geometry moves every step
            sc_t = ctx.scene(scene.data, "spectrum")
            cond_t = _cond_for(capi, ctx, sc_t)
        tr = capi.Trainer(ctx, sc_t, cond_t, hyper, geometry=geometry)
        gbuf = tr.grad_tensor()

        def step():
            # joint: build_tx_state every step from the current geometry (trainer.cpp:417-421)
            st_s = sc_t.tx_state(np.array(TX), grid) if geometry else st
            tr.grads(st_s, rx_d, targets)
            allreduce_grads(gbuf)  # NCCL over NVLink (no-op at world 1)
            tr.apply()

        for _ in range(2):
            step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        n_steps = max(3, min(args.steps, 10))
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(n_steps):
            step()
        s1.record(stream)
        torch.cuda.synchronize(dev)
        return max_over_ranks(s0.elapsed_time(s1) / n_steps, dev), tr.n

    ms, n_grad = time_trainer(list(capi.Trainer.L1_ONLY))  # spectrum L1 (lambda_ssim = lambda_fft = 0)
    hp = list(capi.Trainer.DEFAULTS)
    hp[3], hp[4] = 0.2, 0.1  # the reference's default LossWeights (trainer.hpp:25-29)
    ms_full, _ = time_trainer(hp)
    ms_joint, n_joint = time_trainer(list(capi.Trainer.L1_ONLY), geometry=True)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:  # reference CPU training sample (oracle/_ref), one sample, all host threads in render/backward
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O
            chk = O.reference()
            sc = chk.synth_scene(args.gaussians, 2, 1, 7)
            h = chk.scene(sc, "spectrum")
            lo, hi = chk.scene_bounds(h, 0.0)
            cfg = O.cond_cfg()
            params = chk.synth_cond(cfg, 2, 1, lo, hi, 3, True)
            olo, ohi = chk.scene_bounds(h, 0.1)
            rc = chk.cond(cfg, params, chk.build_occupancy(h, 32, olo, ohi), olo, ohi)
            og = O.Grid(args.n_theta, args.n_phi, 8, 1.0)
            t0 = time.perf_counter()
            chk.train_sample(h, rc, og, TX, rx[0], targets[0].cpu().numpy().astype(np.float64))
            secs = time.perf_counter() - t0
            cpu = {"samples_per_s": 1.0 / secs, "cores": os.cpu_count(), "kind": "reference",
                   "sample": "1 (tx, rx) sample: build_tx_state + condition_forward + render_field + "
                             "composite_loss + aggregate/render/conditioning adjoints (render threads = nproc)"}
        except Exception as ex:
            cpu = {"error": str(ex)}
    return {"workload": f"config4: K={args.gaussians} Stage-II step, {B} (tx, rx) samples per GPU, spectrum L1, "
                        f"conditioning + compositing forward/backward, Adam; f64 gradient all-reduce "
                        f"({'NCCL' if world > 1 else 'none at 1 GPU'}) of {n_grad} values",
            "ms_per_step": ms, "steps_per_s": 1e3 / ms, "samples_per_s": world * B * 1e3 / ms,
            "default_loss": {"lambda_ssim": 0.2, "lambda_fft": 0.1, "ms_per_step": ms_full,
                             "samples_per_s": world * B * 1e3 / ms_full},
            "joint": {"what": "train_joint step: + build_tx_state per step, FP64 backward_render geometry "
                              "gradients, degree mask, Adam on position/transmittance/scaling/rotation",
                      "ms_per_step": ms_joint, "samples_per_s": world * B * 1e3 / ms_joint, "grad_floats": n_joint},
            "grad_floats": n_grad, "n_gpus": world, "cpu_reference": cpu}


def _cond_for(capi, ctx, scene, lib=None):
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg()
    params = capi.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    cond = ctx.cond(cfg, params)
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    return cond


def _ref_model(O, chk, k):
    sc = chk.synth_scene(k, 2, 1, 7)
    h = chk.scene(sc, "spectrum")
    lo, hi = chk.scene_bounds(h, 0.0)
    cfg = O.cond_cfg()
    params = chk.synth_cond(cfg, 2, 1, lo, hi, 3, True)
    olo, ohi = chk.scene_bounds(h, 0.1)
    return h, chk.cond(cfg, params, chk.build_occupancy(h, 32, olo, ohi), olo, ohi)


def bench_coverage(args, capi, ctx, stream, dev, rank, world):
    """BASELINE config 3: RSSI coverage table, K=500k, 64 Tx x 1024 Rx, 90x360.
    The table is split over a gt x gr grid of ranks (dist.coverage_grid:
    transmitter blocks x receiver blocks by a cost model), so per-Tx state
    builds are not replicated on every rank (strong scaling of the fixed
    table).  One step = this rank's block through rxgs_coverage_table:
    global + local conditioning once per receiver (Tx-independent, cached in
    HBM), then per Tx build_tx_state + factorised signal + RSSI compositing.
    Timed with per-kernel profiling OFF; phases come from a separate pass."""
    import torch
    from paper_2605_24290_b200.dist import coverage_grid, coverage_shard, max_over_ranks
    K, n_tx, n_rx_total = 500_000, 64, 1024
    gt, gr = coverage_grid(n_tx, n_rx_total, world)
    tb, te, rb, re_ = coverage_shard(n_tx, n_rx_total, rank, world, (gt, gr))
    rx = capi.synth_points(n_rx_total, 11, "bench.rx", BOX_LO, BOX_HI, 0.05)[rb:re_]
    tx = capi.synth_points(n_tx, 13, "bench.tx", BOX_LO, BOX_HI, 0.05)[tb:te]
    scene = ctx.scene(capi.synth_scene(K, 2, 1, 7), "rssi")
    cond = _cond_for(capi, ctx, scene)
    grid = capi.Grid(90, 360, 8, 1.0)
    rx_d, tx_d = torch.from_numpy(rx).to(dev), torch.from_numpy(tx).to(dev)
    out_d = torch.empty((tx.shape[0], rx.shape[0]), dtype=torch.float32, device=dev)
    n_steps = max(2, min(args.steps, 3))
    scene.coverage_table(cond, grid, tx_d, rx_d, out_d)  # warm-up (pool, caches)
    torch.cuda.synchronize(dev)
    l0 = ctx.launch_count()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(n_steps):
        scene.coverage_table(cond, grid, tx_d, rx_d, out_d)
    s1.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(s0.elapsed_time(s1) / n_steps, dev)
    launches = (ctx.launch_count() - l0) // n_steps
    ctx.reset_stats()  # per-phase times: a separate profiled pass
    ctx.profile(True)
    scene.coverage_table(cond, grid, tx_d, rx_d, out_d)
    torch.cuda.synchronize(dev)
    phases = {n: ctx.kernel_stats(n)[0] for n in ("cond_global", "local_cache", "tx_prep", "sort", "walk",
                                                   "cov_signal", "composite")}
    ctx.profile(False)
    # end to end with host buffers (tx/rx in, table out): one untimed call
    # (first use of the host-buffer path: lazy module loads, staging buffers),
    # then the mean of two timed calls
    out_h = np.empty((tx.shape[0], rx.shape[0]), np.float32)
    scene.coverage_table(cond, grid, tx, rx, out_h)
    torch.cuda.synchronize(dev)
    n_e2e = 2
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        scene.coverage_table(cond, grid, tx, rx, out_h)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / n_e2e, dev)
    queries = n_tx * n_rx_total
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O  # cpu_baseline leg
            chk = O.reference()
            h, rc = _ref_model(O, chk, K)
            s_tx, s_rx, threads = 2, 16, os.cpu_count() or 1
            secs, _, ph = chk.bench_coverage(h, rc, O.Grid(90, 360, 8, 1.0), tx[:s_tx], rx[:s_rx], threads)
            full = ph[0] / s_rx * n_rx_total + ph[1] / s_tx * n_tx + ph[2] / (s_tx * s_rx) * queries
            cpu = {"value": queries / full, "unit": "queries/s", "cores": threads, "kind": "reference",
                   "sample": f"{s_tx} Tx x {s_rx} Rx timed ({secs:.1f} s wall: conditioning {ph[0]:.1f} s, "
                             f"build_tx_state {ph[1]:.1f} s, render+RSSI {ph[2]:.1f} s), extrapolated linearly to "
                             f"64 Tx x 1024 Rx with conditioning once per Rx (BASELINE.md config-3 rule)",
                   "est_table_s": full}
        except Exception as ex:
            cpu = {"error": str(ex)}
    del scene, cond
    ctx.release_cache()
    return {"workload": "config3: K=500k, 64 Tx x 1024 Rx RSSI coverage table, 90x360, conditioned (full)",
            "value": queries / (ms / 1e3), "unit": "queries/s", "ms_per_table": ms, "steps": n_steps,
            "scaling": "strong (fixed table split over ranks)", "n_gpus": world,
            "rank_grid": {"tx_blocks": gt, "rx_blocks": gr, "rank0_block": [tb, te, rb, re_]},
            "e2e": {"value": queries / (e2e_ms / 1e3), "unit": "queries/s", "ms_per_table": e2e_ms,
                    "h2d_bytes_per_step": int(tx.nbytes + rx.nbytes), "d2h_bytes_per_step": int(out_h.nbytes)},
            "phase_ms": phases, "gpu_launches": int(launches), "cpu_baseline": cpu}


def bench_large(args, capi, ctx, stream, dev, rank, world):
    """BASELINE config 5: K=2M, 180x720 (2,070 tiles), 256 Rx per rank, 1 Tx,
    spectrum + RSSI: stress of the sort and the compositor."""
    import torch
    from paper_2605_24290_b200.dist import max_over_ranks, shard_range
    K, n = 2_000_000, 256
    b, e = shard_range(world * n, rank, world)
    rx = capi.synth_points(world * n, 11, "bench.rx", BOX_LO, BOX_HI, 0.05)[b:e]
    scene = ctx.scene(capi.synth_scene(K, 2, 1, 7), "spectrum")
    cond = _cond_for(capi, ctx, scene)
    grid = capi.Grid(180, 720, 8, 1.0)
    tx = np.array(TX)
    rx_d = torch.from_numpy(rx).to(dev)
    spec = torch.empty((n, 180, 720), dtype=torch.float32, device=dev)
    rssi = torch.empty(n, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        st = scene.tx_state(tx, grid)
        scene.render_queries(cond, st, rx_d, spec, rssi)
        return st

    last = None
    for _ in range(2):
        last = step()
    torch.cuda.synchronize(dev)
    n_steps = max(3, min(args.steps, 5))
    l0 = ctx.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]
    for i in range(n_steps):
        flush.fill_(float(i))
        evs[i][0].record(stream)
        last = step()
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / n_steps, dev)
    launches = (ctx.launch_count() - l0) // n_steps
    ctx.reset_stats()  # per-phase times from a separate profiled pass
    ctx.profile(True)
    for i in range(2):
        flush.fill_(float(i))
        last = step()
    torch.cuda.synchronize(dev)
    phases = {nm: ctx.kernel_stats(nm)[0] / 2 for nm in ("tx_prep", "sort", "walk", "cond_global",
                                                        "cond_signal", "composite")}
    ctx.profile(False)
    stats = last.stats()
    del last
    spec_h = torch.empty((n, 180, 720), dtype=torch.float32).pin_memory().numpy()
    rssi_h = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
    rx_h = torch.from_numpy(rx.copy()).pin_memory().numpy()
    st = scene.tx_state(tx, grid)  # warm the host-buffer path
    scene.render_queries(cond, st, rx_h, spec_h, rssi_h)
    del st
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    st = scene.tx_state(tx, grid)
    scene.render_queries(cond, st, rx_h, spec_h, rssi_h)
    del st
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O  # cpu_baseline leg
            chk = O.reference()
            h, rc = _ref_model(O, chk, K)
            threads, sample = os.cpu_count() or 1, 2
            secs, _, _ = chk.bench_queries(h, rc, O.Grid(180, 720, 8, 1.0), TX, rx[:sample], threads)
            cpu = {"value": sample / secs, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{sample} receivers, build_tx_state + conditioning + render + aggregation, "
                             f"{secs:.1f} s wall"}
        except Exception as ex:
            cpu = {"error": str(ex)}
    del scene, cond
    ctx.release_cache()
    return {"workload": "config5: K=2M, 1 Tx x 256 Rx per rank, 180x720 spectrum + RSSI, conditioned (full)",
            "value": world * n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": n_steps, "scaling": "weak",
            "n_gpus": world, "l2": "flushed between timed steps",
            "e2e": {"value": world * n / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(rx.nbytes + 24), "d2h_bytes_per_step": int(spec_h.nbytes + rssi_h.nbytes)},
            "phase_ms": phases, "gpu_launches": int(launches), "tx_state": stats, "cpu_baseline": cpu}


def bench_config1(args, capi, ctx, dev):
    """BASELINE config 1 (the reference's CPU-runnable case): 10k Gaussians,
    1 Tx, 1 Rx = (1.1, 0.7, 0.2), 90x360 spectrum.  Latency of one query end
    to end through the public API (build_tx_state + render_queries with host
    input and output, conditioned), median of 20 after warm-up, wall clock
    around the synchronous calls; rank 0 only (a single query does not shard)."""
    import time
    K = 10_000
    scene = ctx.scene(capi.synth_scene(K, 2, 1, 7), "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg()
    cond = ctx.cond(cfg, capi.synth_cond(cfg, 2, 1, lo, hi, 3, True))
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(args.n_theta, args.n_phi, 8, 1.0)
    tx = np.array(TX)
    rx = np.array([[1.1, 0.7, 0.2]])
    spec = np.empty((1, args.n_theta, args.n_phi), np.float32)
    rssi = np.empty(1, np.float32)

    def query():
        st = scene.tx_state(tx, grid)
        scene.render_queries(cond, st, rx, spec, rssi)

    for _ in range(5):
        query()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        query()
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.median(ts))
    cpu = None
    if not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O  # cpu_baseline leg
            chk = O.reference()
            sc = chk.synth_scene(K, 2, 1, 7)
            h = chk.scene(sc, "spectrum")
            rlo, rhi = chk.scene_bounds(h, 0.0)
            rcfg = O.cond_cfg()
            params = chk.synth_cond(rcfg, 2, 1, rlo, rhi, 3, True)
            rolo, rohi = chk.scene_bounds(h, 0.1)
            rc = chk.cond(rcfg, params, chk.build_occupancy(h, 32, rolo, rohi), rolo, rohi)
            threads = os.cpu_count() or 1
            secs, _, _ = chk.bench_queries(h, rc, O.Grid(args.n_theta, args.n_phi, 8, 1.0), TX, rx, threads)
            cpu = {"ms_per_query": secs * 1e3, "cores": threads, "kind": "reference",
                   "sample": "the same query: build_tx_state + condition_forward + render_field + aggregation"}
        except Exception as ex:
            cpu = {"error": str(ex)}
    del scene, cond
    return {"workload": "config1: K=10k, 1 Tx, 1 Rx (1.1, 0.7, 0.2), 90x360 spectrum + RSSI, conditioned (full)",
            "ms_per_query": ms, "queries_per_s": 1e3 / ms, "what": "wall clock of the synchronous public-API "
            "calls with host buffers (latency-bound: one receiver)", "cpu_reference": cpu}


def bench_lmax9(args, capi, ctx, stream, dev, rank, world):
    """Config 2 at the paper's spectrum setting l_max = 9 (L = 100 FLE
    components; SURVEY.md 8d secondary point)."""
    import torch
    from paper_2605_24290_b200.dist import max_over_ranks, shard_range
    K, n, l_max = args.gaussians, args.rx, 9
    b, e = shard_range(world * n, rank, world)
    rx = capi.synth_points(world * n, 11, "bench.rx", BOX_LO, BOX_HI, 0.05)[b:e]
    scene = ctx.scene(capi.synth_scene(K, l_max, 1, 7), "spectrum")
    lo, hi = scene.bounds(0.0)
    cfg = capi.cond_cfg(l_max=l_max)
    cond = ctx.cond(cfg, capi.synth_cond(cfg, l_max, 1, lo, hi, 3, True))
    olo, ohi = scene.bounds(0.1)
    cond.build_occupancy(scene, 32, olo, ohi)
    grid = capi.Grid(args.n_theta, args.n_phi, 8, 1.0)
    tx = np.array(TX)
    rx_d = torch.from_numpy(rx).to(dev)
    spec = torch.empty((n, args.n_theta, args.n_phi), dtype=torch.float32, device=dev)
    rssi = torch.empty(n, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        st = scene.tx_state(tx, grid)
        scene.render_queries(cond, st, rx_d, spec, rssi)
        return st

    last = None
    for _ in range(2):
        last = step()
    torch.cuda.synchronize(dev)
    n_steps = max(3, min(args.steps, 5))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]
    for i in range(n_steps):
        flush.fill_(float(i))
        evs[i][0].record(stream)
        last = step()
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / n_steps, dev)
    ctx.reset_stats()
    ctx.profile(True)
    last = step()
    torch.cuda.synchronize(dev)
    phases = {nm: ctx.kernel_stats(nm)[0] for nm in ("tx_prep", "sort", "walk", "cond_global", "cond_signal",
                                                    "composite")}
    ctx.profile(False)
    del last
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O  # cpu_baseline leg
            chk = O.reference()
            sc = chk.synth_scene(K, l_max, 1, 7)
            h = chk.scene(sc, "spectrum")
            rlo, rhi = chk.scene_bounds(h, 0.0)
            rcfg = O.cond_cfg(l_max=l_max)
            params = chk.synth_cond(rcfg, l_max, 1, rlo, rhi, 3, True)
            rolo, rohi = chk.scene_bounds(h, 0.1)
            rc = chk.cond(rcfg, params, chk.build_occupancy(h, 32, rolo, rohi), rolo, rohi)
            threads, sample = os.cpu_count() or 1, 8
            secs, _, _ = chk.bench_queries(h, rc, O.Grid(args.n_theta, args.n_phi, 8, 1.0), TX, rx[:sample], threads)
            cpu = {"value": sample / secs, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{sample} receivers, build_tx_state + conditioning + render + aggregation, "
                             f"{secs:.1f} s wall"}
        except Exception as ex:
            cpu = {"error": str(ex)}
    del scene, cond
    ctx.release_cache()
    return {"workload": f"config2 at l_max=9: K={K}, 1 Tx x {n} Rx per rank, {args.n_theta}x{args.n_phi}, "
                        f"L=100 FLE components, spectrum + RSSI, conditioned (full)",
            "value": world * n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": n_steps, "scaling": "weak",
            "n_gpus": world, "l2": "flushed between timed steps", "phase_ms": phases, "cpu_baseline": cpu}


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the path
    (oracle/_ref) on all host threads, rank 0 only.  Each step is a bounded
    sample of the config-2 step: build_tx_state + 256 of its 1024 receivers."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or 256
    setup = cpu_reference_setup(args)
    for _ in range(min(args.warmup, 1)):
        cpu_reference_run(args, min(sample, 4), threads, setup)
    t = []
    for _ in range(args.steps):
        secs, kind = cpu_reference_run(args, sample, threads, setup)
        t.append(secs)
    v = sample / (sum(t) / len(t))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(t) / len(t), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(args), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "cpu_model": cpu_model(),
                             "sample": f"{sample} receivers per step of the same workload (build_tx_state once "
                                       f"per step + condition_forward fanned over {threads} threads + "
                                       f"render_field chunks of 16 with threads={threads} + aggregation)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command under
    torch.distributed.run, one rank (process) per GPU on 127.0.0.1; rank 0
    prints the JSON line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
