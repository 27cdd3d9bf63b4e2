"""bench.py -- NTBC inference hot path on B200: BC blocks decoded/s and ms per 4k material.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

A step = one pass of the whole hot path over synthetic 4k materials (config
C3: 4096^2, diffuse+normal BC1, roughness+AO+displacement BC4 -- MetalPlates013-shaped), one
ntbc_decode_material call per material (grid dequant launch + fused-kernel launch).  N = 1: one material
per step (the metric's "ms per 4k material").  N > 1 (torchrun): BASELINE config 5, a batch of 64 C3-shaped
materials (distinct seeds) sharded 64/N per rank (--materials), every rank's fused kernel storing its BC
words straight into rank 0's buffer (the final gather of packed bytes, counted in the timing; north_star).
Rank 0 prints ONE JSON line.

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
def pack_roofline(model, spec, W, H, dev, peaks, reps=20):
    """Kernel (2) standalone (ntbc_pack, rows a5-a8 fed the fp32 MLP outputs of the whole C3 material, produced
    once by ntbc_debug_mlp): HBM roofline.  Algorithmic bytes per launch = the fp32 endpoint + colour outputs
    read once + the BC words written once."""
    import torch

    from paper_2407_09543_b200 import ntbc
    fmts = list(spec.fmts)
    ep_d, col_d = ntbc.debug_mlp(model, W, H)
    outs = [torch.empty((H // 4, W // 4), dtype=torch.int64, device=dev) for _ in fmts]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        ntbc.pack(fmts, ep_d, col_d, W, H, outs=outs)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ntbc.pack(fmts, ep_d, col_d, W, H, outs=outs)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sum(ts) / len(ts)
    nbytes = ep_d.numel() * 4 + col_d.numel() * 4 + len(fmts) * (W // 4) * (H // 4) * 8
    peak = peaks.get("hbm_gbs", 6556.2)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_pack_traffic.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    return {"kernel": f"pack_kernel<{len(fmts)}>", "bound": "hbm", "achieved": nbytes / (ms * 1e-3) / 1e9,
            "peak": peak, "unit": "GB/s", "frac": nbytes / (ms * 1e-3) / 1e9 / peak, "traffic": traffic,
            "bytes_per_launch": nbytes, "kernel_ms": ms,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2407_09543_b200 import ntbc
    from paper_2407_09543_b200.shard import PeerGather, PeerRows, gather_materials, material_shards

    # NTBC_BENCH_ONE_GPU=1: functional check of the multi-rank path on a one-GPU box (every rank on cuda:0,
    # gloo process group; the ranks' kernels never wait on each other).  Its numbers are not measurements.
    if os.environ.get("NTBC_BENCH_ONE_GPU") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W, H, spec = synth.config_shape(args.config)
    n_mat = args.materials or (1 if world == 1 else 64)
    lo, hi = material_shards(n_mat, world)[rank]
    blobs = [synth.model_blob(args.config, material=g) for g in range(lo, hi)]
    models = [ntbc.Model(b, local_rank) for b in blobs]
    n_tex = len(spec.fmts)
    BW, BH = W // 4, H // 4
    plane = BH * BW
    out_all = torch.empty((max(1, hi - lo), n_tex, BH, BW), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()
    # the final gather of packed bytes to rank 0 (north star), inside the timed step: fused into the decode
    # by default (every rank's kernel stores its BC words into rank 0's buffer over NVLink, PeerGather);
    # NTBC_GATHER=nccl uses a separate NCCL gather after the decode instead
    gather_mode = os.environ.get("NTBC_GATHER", "peer") if world > 1 else "none"
    pg = PeerGather(n_tex, BH, BW, rank, world, dev, n_materials=n_mat) if gather_mode == "peer" else None
    if pg is not None and not pg.ok:   # no IPC / peer access on this system: all ranks fall back together
        print(f"rank {rank}: peer gather unavailable ({pg.error}); using the NCCL gather", file=sys.stderr)
        pg.close()
        pg, gather_mode = None, "nccl"
    if gather_mode == "nccl" and len({e - b for b, e in material_shards(n_mat, world)}) != 1:
        raise SystemExit("--materials must be a multiple of the world size for the NCCL gather")

    def step():
        for i, m in enumerate(models):
            if pg is not None:
                ntbc.decode_material([m], W, H, out_ptrs=pg.ptrs_of(lo + i), stream=stream)
            else:
                ntbc.decode_material([m], W, H, outs=[out_all[i, k] for k in range(n_tex)], stream=stream)
        if pg is not None:
            pg.complete()
        elif world > 1:
            for i in range(hi - lo):
                gather_materials(out_all[i], rank, world)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ntbc.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # the dominant kernel (fused_decode_kernel) timed live inside the timed steps: the library records these
    # events right before / after each fused launch on the launch stream (ntbc_debug_time_fused); with several
    # materials per step the pair holds the step's last launch
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:   # torch creates the CUDA events lazily on first record
        a.record(stream)
        b.record(stream)
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for s_ in range(args.steps):
            flush.zero_()                                  # L2 flushed between timed steps (not timed)
            ntbc.time_fused(*kev[s_])
            evs[s_][0].record(stream)
            step()
            evs[s_][1].record(stream)
        torch.cuda.synchronize()
    ntbc.time_fused(None, None)
    if world > 1:
        dist.barrier()
    launches = ntbc.launch_count() - launches0
    if pg is not None and rank == 0:   # rank 0's buffer holds every rank's materials: spot-check our first one
        ntbc.decode_material([models[0]], W, H, outs=[out_all[0, k] for k in range(n_tex)], stream=stream)
        torch.cuda.synchronize()
        assert torch.equal(pg.buf[lo], out_all[0]), "peer gather: rank 0 slice differs from a local decode"
    times = [a.elapsed_time(b) for a, b in evs]
    t_ms = sum(times) / len(times)
    k_ms = sum(a.elapsed_time(b) for a, b in kev) / len(kev)

    # ---- latency view (N > 1, peer gather): ONE material split by block rows over the ranks, every rank
    # decoding its rows straight into rank 0's buffer; time = max over ranks (the metric's "ms per 4k
    # material at N GPUs" as a single-material latency, beside the batch throughput above)
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
    t_tensor = torch.tensor([t_ms, k_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_ms_max, k_ms_max = (float(x) for x in t_tensor.tolist())

    # ---- the other arithmetic contracts on the same material (fused kernel only, timed like k_ms):
    # F (binary32 activations, hi/lo split MMA operands) -- the contract under which the
    # decode meets north_star's rule literally against the plain definitions; P (the hidden selu in binary16
    # arithmetic on f16x2 lanes) -- faster, further from the plain definitions
    def time_contract(c):
        ntbc.set_contract(models[0], c)
        for _ in range(3):
            ntbc.decode_material([models[0]], W, H, outs=[out_all[0, k] for k in range(n_tex)], stream=stream)
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a, b in fev:
            a.record(stream)
            b.record(stream)
        for a, b in fev:
            flush.zero_()
            ntbc.time_fused(a, b)
            ntbc.decode_material([models[0]], W, H, outs=[out_all[0, k] for k in range(n_tex)], stream=stream)
        torch.cuda.synchronize()
        ntbc.time_fused(None, None)
        ntbc.set_contract(models[0], 0)
        fk = sum(a.elapsed_time(b) for a, b in fev) / len(fev)
        return {"kernel_ms": fk, "mblocks_per_s": plane * n_tex / (fk * 1e-3) / 1e6}

    contract_f = contract_p = None
    if world == 1:
        contract_f = dict(time_contract(1), note="fused kernel under ntbc_set_contract(m, 1); the headline value "
                                                 "uses the paper's binary16 contract H")
        contract_p = dict(time_contract(2), note="fused kernel under ntbc_set_contract(m, 2): selu in binary16 "
                                                 "arithmetic (~21% of activations not correctly rounded, §8.f2)")

    # ---- end to end through the C ABI with host buffers (pinned blob in, pinned BC words out), per rank
    model, blob = models[0], blobs[0]
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
    for s_ in range(e_steps):
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
    blocks_step = plane * n_tex * n_mat
    value = blocks_step / (t_ms_max * 1e-3) / 1e6
    clocks = clk.summary()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    sm_now = clocks.get("sm_mhz") or sm_max
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # roofline of the dominant kernel: algorithmic MLP FLOPs per launch (2 x MACs of the paper's
    # layers, unpadded: 333,824 per C3 block position x 1,048,576 positions) / fused-kernel time, against the
    # measured dense 16-bit tensor peak (fp16 = bf16 rate on B200; burst figure: the kernel is timed alone)
    flops = mma_flops_per_material(spec, W, H)
    t_peak = peaks.get("bf16_tflops", 1691.9)
    achieved = flops / (k_ms_max * 1e-3) / 1e12
    traffic, ncu_ctx, issue = None, None, None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_fused_traffic.json")))
        if prof.get("config") == args.config:
            traffic = prof.get("dram_bytes_per_launch")
            ncu_ctx = {k: prof.get(k) for k in ("source", "issue_active", "alu_pipe", "fma_pipe", "tensor_pipe",
                                                 "thread_instructions_per_texel")}
            ipt = prof.get("thread_instructions_per_texel")
            if ipt:
                # the binding resource: SIMT issue.  SASS thread-instructions per texel (ncu, committed capture)
                # x texels / (SMs x 128 lanes x SM clock under load x live fused-kernel time)
                cap = n_sm * 128 * sm_now * 1e6 * k_ms_max * 1e-3
                issue = {"thread_instructions_per_texel": ipt, "texels": W * H,
                         "frac": ipt * W * H / cap, "sm_mhz": sm_now,
                         "definition": "ncu SASS thread-instructions/texel x texels / (SMs x 128 x clock x kernel time)"}
    except Exception:
        pass
    hbm_bytes = len(blob) + plane * n_tex * 8
    pack = None
    if world == 1 and not args.no_pack:
        pack = pack_roofline(models[0], spec, W, H, dev, peaks)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu, _, _ = oracle_sample(args.config, budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms_max, "higher_is_better": True,
        "scaling": "weak" if n_mat == world else "strong",
        "vs_baseline": None, "dtype": "f16 MMA operands / f32 accumulate+epilogue", "data": "synthetic",
        "config": {"workload": synth.CONFIGS[args.config]["name"] if n_mat == 1 else
                   f"C5: batch of {n_mat} x " + synth.CONFIGS[args.config]["name"],
                   "width": W, "height": H,
                   "textures": len(spec.fmts), "formats": ["BC1" if f == 1 else "BC4" for f in spec.fmts],
                   "model": "paper architecture (P:330-343), random-init seeded weights",
                   "materials_per_step": n_mat, "materials_per_rank": hi - lo, "gather_to_rank0": world > 1,
                   "gather": {"none": None, "peer": "fused: each rank's kernel stores its BC words into rank 0's "
                              "buffer over NVLink (CUDA IPC), completion by a 1-element all-reduce",
                              "nccl": "separate NCCL gather after the decode"}[gather_mode],
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "ms_per_4k_material": t_ms_max * world / n_mat,
                   "latency_ms_per_4k_material": lat_ms if world > 1 else t_ms_max,
                   "contract": "H (binary16 MMA operands at every layer input, P:322)",
                   "contract_f": contract_f, "contract_p": contract_p},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": t_peak, "unit": "TFLOP/s",
                     "frac": achieved / t_peak, "traffic": traffic,
                     "kernel": "fused_decode_kernel", "kernel_ms": k_ms_max,
                     "flops_per_launch": flops, "flops_per_block_position": flops // plane,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; dense fp16 = bf16 rate)",
                     "issue": issue,
                     "hbm": {"bytes_per_launch": hbm_bytes, "achieved_gbs": hbm_bytes / (k_ms_max * 1e-3) / 1e9,
                             "frac": hbm_bytes / (k_ms_max * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6556.2)},
                     "ncu": ncu_ctx, "pack": pack},
        "cpu_baseline": cpu,
        "e2e": {"value": plane * n_tex * world / (e_ms * 1e-3) / 1e6, "unit": UNIT, "ms_per_step": e_ms,
                "h2d_bytes_per_step": len(blob) * world, "d2h_bytes_per_step": plane * n_tex * 8 * world,
                "api": "ntbc_decode_material_host (pinned host blob -> device -> BC words -> pinned host), "
                       "one material per rank per step"},
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
    ap.add_argument("--materials", type=int, default=None,
                    help="materials per step over all ranks (default: 1 at N = 1, BASELINE config 5's 64 at N > 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pack", action="store_true", help="skip the standalone pack kernel's HBM roofline")
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
