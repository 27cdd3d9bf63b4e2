"""bench.py -- NTBC inference hot path on B200: BC blocks decoded/s and ms per 4k material.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

A step = one pass of the whole hot path over one synthetic 4k material
(config C3: 4096^2, diffuse+normal BC1, roughness+AO+displacement BC4 -- MetalPlates013-shaped),
i.e. one ntbc_decode_material call (one fused-kernel launch).  Under torchrun (N>1) every rank
decodes its own material (weak scaling) and the packed BC bytes are gathered to rank 0 with NCCL
inside the timed region (BASELINE.json north_star: "only a final gather of packed bytes, counted in
the timing").  Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (the reference arm for this paper-only task)
on a bounded sample of block rows per step, on this box's host cores.
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

METRIC = "BC blocks decoded/sec and ms per 4k material at 1/2/4/8 B200 (% roofline)"
UNIT = "Mblocks/s"


# ---------------------------------------------------------------- algorithmic work model
def ops_per_material(spec, W, H):
    """Algorithmic element-wise ops of the pinned definitions (R6, R8, R9, R11-R18), excluding the
    tensor-core contraction: one op per IEEE operation, integer op or conversion."""
    n_bc1 = sum(1 for f in spec.fmts if f == 1)
    n_bc4 = len(spec.fmts) - n_bc1
    # per hidden activation (incl. fp16 cvt, R9 v3), per sigmoid, per grid level and texel (coordinates, floor,
    # fractions, index, 3 lerps x 2 features, fp16 cvt; the Eq.2 dequantization runs once per vertex in
    # dequant_grids_kernel since r01w and is not counted per texel)
    selu, sig, lvl = 18, 16, 22
    hidden = spec.hidden * spec.n_hidden
    per_texel = hidden * selu + spec.n_color_out * sig + spec.texel_levels * lvl + 4 + 46 * n_bc1 + 42 * n_bc4
    per_block = (hidden * selu + spec.n_endpoint_out * sig + spec.block_levels * lvl + 4 + 40 * n_bc1 + 12 * n_bc4)
    blocks = (W // 4) * (H // 4)
    return blocks * (16 * per_texel + per_block), per_texel, per_block


def mma_flops_per_material(spec, W, H):
    """Algorithmic MLP FLOPs (2 x MACs of the paper's layers, unpadded)."""
    def macs(dims):
        return sum(a * b for a, b in zip(dims[:-1], dims[1:]))
    blocks = (W // 4) * (H // 4)
    return 2 * blocks * (16 * macs(spec.mlp_dims("color")) + macs(spec.mlp_dims("endpoint")))


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

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
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU oracle timing (baseline / reference arm)
def oracle_sample(cfg: int, budget_s: float = 15.0, material: int = 0):
    """Time the oracle, as it stands, on a bounded sample of full-width block rows of the workload."""
    import oracle
    import synth
    W, H, spec = synth.config_shape(cfg)
    om = oracle.Model(synth.model_blob(cfg, material))
    threads = os.cpu_count() or 1
    om.decode_material(W, H, 0, 1, nthreads=threads)          # warm-up (thread pool, page-in)
    est = max(1, min(threads, H // 8))                        # the oracle parallelises over rows: estimate
    t0 = time.perf_counter()                                  # the per-row cost with every thread busy
    om.decode_material(W, H, 1, 1 + est, nthreads=threads)
    t_row = (time.perf_counter() - t0) / est
    r0 = 1 + est
    rows = int(max(1, min(H // 4 - r0, budget_s / max(t_row, 1e-3))))
    t0 = time.perf_counter()
    om.decode_material(W, H, r0, r0 + rows, nthreads=threads)
    dt = time.perf_counter() - t0
    blocks = rows * (W // 4) * len(spec.fmts)
    return {"value": blocks / dt / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{rows} full-width block rows ({rows * (W // 4)} block positions x {len(spec.fmts)} "
                      f"textures) of the {W}x{H} material, {dt:.1f}s"}, om, rows


def run_reference(args, rank, world):
    import synth
    if rank != 0:
        return
    W, H, spec = synth.config_shape(args.config)
    import oracle
    om = oracle.Model(synth.model_blob(args.config))
    threads = os.cpu_count() or 1
    # each step: one full-width block row per host thread (the oracle parallelises over rows), about
    # 2 s of host time on 16 cores, so that every core is busy and K steps end within minutes
    rows = max(1, min(threads, H // 4))
    for _ in range(args.warmup):
        om.decode_material(W, H, 0, rows, nthreads=threads)
    t0 = time.perf_counter()
    for s in range(args.steps):
        r0 = (s * rows) % (H // 4)
        om.decode_material(W, H, r0, min(H // 4, r0 + rows), nthreads=threads)
    dt = time.perf_counter() - t0
    blocks = args.steps * rows * (W // 4) * len(spec.fmts)
    value = blocks / dt / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16/f32 (oracle, C99)",
        "data": "synthetic",
        "config": {"workload": synth.CONFIGS[args.config]["name"], "width": W, "height": H,
                   "textures": len(spec.fmts), "step": f"{rows} full-width block row(s) of the material (bounded sample)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{args.steps} steps x {rows} block row(s) x {W // 4} blocks x {len(spec.fmts)} textures"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2407_09543_b200 import ntbc
    from paper_2407_09543_b200.shard import PeerGather, PeerRows, gather_materials

    # NTBC_BENCH_ONE_GPU=1: functional check of the multi-rank path on a one-GPU box (every rank on cuda:0,
    # gloo process group; the ranks' kernels never wait on each other).  Its numbers are not measurements.
    if os.environ.get("NTBC_BENCH_ONE_GPU") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W, H, spec = synth.config_shape(args.config)
    blob = synth.model_blob(args.config, material=rank)
    model = ntbc.Model(blob, local_rank)
    n_tex = model.n_tex
    BW, BH = W // 4, H // 4
    plane = BH * BW
    out_all = torch.empty((n_tex, BH, BW), dtype=torch.int64, device=dev)   # contiguous for the gather
    outs = [out_all[k] for k in range(n_tex)]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()
    # the final gather of packed bytes to rank 0 (north star), inside the timed step: fused into the decode
    # by default (every rank's kernel stores its BC words into rank 0's buffer over NVLink, PeerGather);
    # NTBC_GATHER=nccl uses a separate NCCL gather after the decode instead
    gather_mode = os.environ.get("NTBC_GATHER", "peer") if world > 1 else "none"
    pg = PeerGather(n_tex, BH, BW, rank, world, dev) if gather_mode == "peer" else None
    if pg is not None and not pg.ok:   # no IPC / peer access on this system: all ranks fall back together
        print(f"rank {rank}: peer gather unavailable ({pg.error}); using the NCCL gather", file=sys.stderr)
        pg.close()
        pg, gather_mode = None, "nccl"

    def step():
        if pg is not None:
            ntbc.decode_material([model], W, H, out_ptrs=pg.ptrs, stream=stream)
            pg.complete()
        else:
            ntbc.decode_material([model], W, H, outs=outs, stream=stream)
            if world > 1:
                gather_materials(out_all, rank, world)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ntbc.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        for s in range(args.steps):
            flush.zero_()                                  # L2 flushed between timed steps (not timed)
            evs[s][0].record(stream)
            step()
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ntbc.launch_count() - launches0
    if pg is not None and rank == 0:   # rank 0's buffer holds every rank's material: spot-check our own slice
        ntbc.decode_material([model], W, H, outs=outs, stream=stream)
        torch.cuda.synchronize()
        assert torch.equal(pg.buf[0], out_all), "peer gather: rank 0 slice differs from a local decode"
    times = [a.elapsed_time(b) for a, b in evs]
    t_ms = sum(times) / len(times)

    # ---- latency view (N > 1, peer gather): ONE material split by block rows over the ranks, every rank
    # decoding its rows straight into rank 0's buffer; time = max over ranks (the metric's "ms per 4k
    # material at N GPUs" as a single-material latency, beside the weak-scaling throughput above)
    lat_ms = None
    if pg is not None:
        pr = PeerRows(n_tex, BH, BW, rank, world, dev)
        if pr.ok:
            model0 = ntbc.Model(synth.model_blob(args.config, material=0), local_rank)   # one material on all ranks

            def lat_step():
                ntbc.decode_material([model0], W, H, row_begin=pr.r0, row_end=pr.r1, out_ptrs=pr.ptrs, stream=stream)
                pr.complete()
            for _ in range(3):
                lat_step()
            torch.cuda.synchronize()
            dist.barrier()
            lev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for s_ in range(args.steps):
                flush.zero_()
                lev[s_][0].record(stream)
                lat_step()
                lev[s_][1].record(stream)
            torch.cuda.synchronize()
            lt = torch.tensor([sum(a.elapsed_time(b) for a, b in lev) / args.steps], device=dev, dtype=torch.float64)
            dist.all_reduce(lt, op=dist.ReduceOp.MAX)
            lat_ms = float(lt.item())
            if rank == 0:   # rank 0's buffer holds the whole material: it must equal a local decode
                ref = torch.stack(ntbc.decode_material([model0], W, H, stream=stream))
                torch.cuda.synchronize()
                assert torch.equal(pr.buf, ref), "row-split peer decode differs from a local decode"
        pr.close()
        dist.barrier()
    t_tensor = torch.tensor([t_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_ms_max = float(t_tensor.item())

    # ---- kernel-only timing of the dominant kernel (the fused decode kernel), same stream
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s in range(args.steps):
        flush.zero_()
        kev[s][0].record(stream)
        ntbc.decode_material([model], W, H, outs=outs, stream=stream)
        kev[s][1].record(stream)
    torch.cuda.synchronize()
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps

    # ---- end to end through the C ABI with host buffers (pinned blob in, pinned BC words out)
    pinned_blob = torch.frombuffer(bytearray(blob), dtype=torch.uint8).pin_memory()
    host_all = torch.empty((n_tex, BH, BW), dtype=torch.int64).pin_memory()   # one pinned [tex][BH][BW] buffer
    host_out = [host_all[k] for k in range(n_tex)]
    for _ in range(2):
        ntbc.decode_material_host([model], [pinned_blob], W, H, host_out, stream=stream)
    torch.cuda.synchronize()
    # consecutive calls pipeline (the next material's upload overlaps the current decode, copy-back
    # overlaps the kernel), so time the whole span of e_steps calls on the device, not per call
    e_steps = max(3, min(args.steps, 20))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(e_steps):
        ntbc.decode_material_host([model], [pinned_blob], W, H, host_out, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1) / e_steps
    e_tensor = torch.tensor([e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e_tensor, op=dist.ReduceOp.MAX)
    e_ms = float(e_tensor.item())
    if pg is not None:   # unmap rank 0's buffer everywhere before rank 0 may free it
        pg.close()
        dist.barrier()

    if rank != 0:
        return
    blocks_step = plane * n_tex * world
    value = blocks_step / (t_ms_max * 1e-3) / 1e6
    ops, per_texel, per_block = ops_per_material(spec, W, H)
    clocks = clk.summary()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = n_sm * 128 * sm_max * 1e6 / 1e9          # Gop/s: 128 lane-instructions / clk / SM
    achieved = ops / (k_ms * 1e-3) / 1e9
    traffic, ncu_ctx = None, None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_fused_traffic.json")))
        if prof.get("config") == args.config:
            traffic = prof.get("dram_bytes_per_launch")
            # cross-check of the op-count fraction with hardware counters from the committed ncu capture
            ncu_ctx = {k: prof.get(k) for k in ("source", "issue_active", "alu_pipe", "fma_pipe", "tensor_pipe",
                                                 "thread_instructions_per_texel")}
    except Exception:
        pass
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu, _, _ = oracle_sample(args.config, budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16 MMA operands / f32 accumulate+epilogue", "data": "synthetic",
        "config": {"workload": synth.CONFIGS[args.config]["name"], "width": W, "height": H,
                   "textures": len(spec.fmts), "formats": ["BC1" if f == 1 else "BC4" for f in spec.fmts],
                   "model": "paper architecture (P:330-343), random-init seeded weights",
                   "materials_per_rank_per_step": 1, "gather_to_rank0": world > 1,
                   "gather": {"none": None, "peer": "fused: each rank's kernel stores its BC words into rank 0's "
                              "buffer over NVLink (CUDA IPC), completion by a 1-element all-reduce",
                              "nccl": "separate NCCL gather after the decode"}[gather_mode],
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "ms_per_4k_material": t_ms_max / world if world > 1 else t_ms_max,
                   "latency_ms_per_4k_material": lat_ms if world > 1 else t_ms_max},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "Gop/s",
                     "frac": achieved / alu_peak, "traffic": traffic,
                     "kernel": "fused_decode_kernel", "kernel_ms": k_ms,
                     "kernel_ms_covers": "CUDA events around ntbc_decode_material: dequant_grids_kernel "
                                         "(row a2's Eq.2 half, ~1% of the step) + fused_decode_kernel",
                     "ops_per_texel": per_texel, "ops_per_block": per_block, "ncu": ncu_ctx,
                     "peak_source": f"{n_sm} SMs x 128 lane-instr/clk x {sm_max:.0f} MHz (DESIGN.md §7.3)",
                     "tensor": {"achieved_tflops": mma_flops_per_material(spec, W, H) / (k_ms * 1e-3) / 1e12,
                                "peak_tflops": peaks.get("bf16_tflops", 1658.0),
                                "frac": mma_flops_per_material(spec, W, H) / (k_ms * 1e-3) / 1e12 /
                                peaks.get("bf16_tflops", 1658.0)}},
        "cpu_baseline": cpu,
        "e2e": {"value": blocks_step / (e_ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": e_ms,
                "h2d_bytes_per_step": len(blob), "d2h_bytes_per_step": plane * n_tex * 8,
                "api": "ntbc_decode_material_host (pinned host blob -> device -> BC words -> pinned host)"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("NTBC_BENCH_ONE_GPU") == "1":   # functional check only (see run_ours)
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
