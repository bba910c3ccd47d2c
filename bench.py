#!/usr/bin/env python3
"""Benchmark of the B200 fractal encoder — BASELINE.json's metric:
range-domain comparisons/sec (and encode ms/image) vs the CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Workload (N=1): cfg2 = BASELINE.json configs[1], a 512x512 synthetic CT slice, 8x8 ranges,
domain stride 4, 8 isometries, full search.  A "step" encodes one image: normalised pool
build (K1), range pass, seed, the tcgen05 scan levels with their exact survivor evaluation
(K2), winner selection and records — with the image resident in HBM (`value`) or through
the public API with host buffers (`e2e`, H2D + D2H inside the timed region).  The roofline
is reported for the dominant kernel (the full-level scan: all R x D x 8 correlations, against
the measured bf16 peak and a measured int8 peak), the pool builder (HBM) and the decoder (HBM).

Multi-GPU (torchrun, one rank per GPU, NCCL), the north_star's splits:
  --config cfg4   one 2048^2 image, its range rows sharded over the ranks (every rank builds the
                  replicated pool, fic_encode_rows_device), records gathered to rank 0 (strong);
  --config cfg5   the 512-slice volume sharded by slices over the ranks, up to 64 slices per
                  encode pass, records gathered to rank 0 (strong);
  cfg1-cfg3       each rank encodes its own image (weak), records gathered to rank 0.
`value` counts every rank's own comparisons (summed) over the max-over-ranks device time.

CPU baseline / --impl reference: the unmodified reference (oracle/_ref) on the host cores:
a full encode_parallel over every thread for cfg1-cfg3 (and one cfg5 slice), best of the
runs; a seeded random range sample via encode_range for cfg4, extrapolated.

The unit of work is one comparison = one (range, domain, isometry) candidate, counted as
EncodeStats.candidates_tested (proj/include/fic/encoder.hpp:50), identical for CPU and GPU.
"""
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

METRIC = "range-domain comparisons/sec and encode ms/image at 1/2/4/8 B200 vs CPU ref"
UNIT = "comparisons/s"
CONFIG_TEXT = {
    "cfg1": "256x256 synthetic phantom, 8x8 ranges, 16x16 domains stride 8, 8 isometries, full search",
    "cfg2": "512x512 CT-slice-shaped synthetic image, 8x8 ranges, domain stride 4, 8 isometries, full search",
    "cfg3": "512x512 synthetic image, 4x4 ranges, 8x8 domains stride 2, 8 isometries, full search",
    "cfg4": "2048x2048 X-ray-shaped synthetic image, 8x8 ranges, domain stride 2, 8 isometries, full search",
    "cfg5": "volume of 512x512 CT-shaped synthetic slices, 8x8 ranges, domain stride 4, 8 isometries, full search, "
            "slices sharded over the ranks, up to 64 slices stacked per encode pass",
}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def make_image(cfg, rank=0, world=1, slices=512):
    """The step's input: one image, or (cfg5) this rank's shard of the slice volume."""
    from paper_1404_0774_b200 import images
    if cfg == "cfg5":
        per = (slices + world - 1) // world
        return images.volume_slices(rank * per, per, slices), 8, 4
    gen, n, step = images.CONFIGS[cfg]
    if rank == 0 or cfg not in ("cfg2", "cfg3"):
        img = gen()
    else:  # weak scaling: each rank its own slice of the cfg5-style volume
        img = images.ct_slice(512, 1404002 + rank, rank / 512.0)
    return img, n, step


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 1590.0, 6650.0, "fallback"


def traffic_for(cfg):
    """dram bytes per matcher launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "matcher_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(cfg)
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- CPU baseline
FULL_CPU = ("cfg1", "cfg2", "cfg3")  # the reference runs these in full


def cpu_reference(cfg, img, n, step, threads, reps, target_ranges=1024, seed=1404):
    """The reference's own encoder (oracle/_ref/libfic_ref.so: the unmodified sources compiled by
    oracle/Makefile with its Release flags) on the box's host cores.

    cfg1-cfg3 (and one cfg5 slice): a FULL encode_parallel(workers = threads, chunk 16x16)
    (proj/src/encoder.cpp:368-427, as proj/tools/bench.cpp:68-74,97-102 runs it), best of `reps`.
    cfg4: encode_range (encoder.cpp:332-342, the identical per-range search) on a seeded random
    sample of `target_ranges` ranges spread over `threads` host threads, best of `reps`,
    extrapolated to the whole image.  Returns a dict with the comparisons/s and the sample."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import Reference
    ref = Reference()
    side = img.shape[0]
    R = (side // n) ** 2
    pv = dict(n=n, step=step)
    times = []
    if cfg in FULL_CPU or cfg == "cfg5":
        for _ in range(reps):
            t0 = time.perf_counter()
            _, st = ref.encode(img, pv, workers=threads, chunk=(16, 16))
            times.append(time.perf_counter() - t0)
        comps = st["candidates_tested"]
        best = min(times)
        sample = (f"full encode_parallel(workers={threads}, chunk 16x16) of " +
                  ("one 512x512 slice of the volume" if cfg == "cfg5" else "the image") + f", best of {reps}")
        return {"value": comps / best, "comparisons": comps, "seconds": best, "all_seconds": times,
                "encode_ms_per_image": best * 1e3, "extrapolated": False, "sample": sample}
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(R, min(target_ranges, R), replace=False))

    def work(chunk):
        c = 0
        for r in chunk:
            _, st = ref.encode_range(img, int(r % (side // n)) * n, int(r // (side // n)) * n, pv)
            c += st["candidates_tested"]
        return c

    chunks = [idx[i::threads] for i in range(threads)]
    for _ in range(reps):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            comps = sum(ex.map(work, chunks))
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"value": comps / best, "comparisons": comps, "seconds": best, "all_seconds": times,
            "encode_ms_per_image": (R / len(idx)) * best * 1e3, "extrapolated": True,
            "sample": f"{len(idx)} of {R} ranges (seeded random) via the reference encode_range over {threads} "
                      f"threads, best of {reps}, extrapolated to the image"}


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    img, n, step = make_image(args.config, slices=1)
    if img.ndim == 3:  # cfg5: the per-slice encode is the unit the reference runs
        img = img[0]
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference(args.config, img, n, step, threads, 1, args.ref_ranges)
    res = cpu_reference(args.config, img, n, step, threads, max(args.steps, 1), args.ref_ranges)
    value = res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic", "config": {"workload": CONFIG_TEXT[args.config], "cfg": args.config, "n": n, "step": step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": res["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "encode_ms_per_image": res["encode_ms_per_image"], "extrapolated": res["extrapolated"],
        "step_seconds": res["all_seconds"],
    }
    print(json.dumps(line), flush=True)
    return 0


def int8_peak_tops():
    """Dense int8 tensor-core throughput of this B200, measured: torch._int_mm (cuBLASLt int8 GEMM)
    at 8192^3, 2 N^3 ops, best of 10 launches timed with CUDA events.  None if unsupported."""
    import torch
    try:
        N = 8192
        a = torch.randint(-64, 64, (N, N), dtype=torch.int8, device="cuda")
        b = torch.randint(-64, 64, (N, N), dtype=torch.int8, device="cuda")
        for _ in range(3):
            torch._int_mm(a, b)
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        return 2.0 * N ** 3 / (best / 1e3) / 1e12
    except Exception:  # noqa: BLE001 — reported as unmeasured
        return None


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1404_0774_b200 as fic
    from paper_1404_0774_b200.sharding import encode_sharded, plan_rows
    from paper_1404_0774_b200.abi import MAPPING_DTYPE

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        args.gpus = world
    # one rank per GPU over NCCL; more ranks than GPUs (a 2-rank check on a 1-GPU box) share
    # devices and exchange over gloo (NCCL refuses two ranks on one device)
    ndev = max(torch.cuda.device_count(), 1)
    dev = local % ndev
    backend = "nccl" if world <= ndev else "gloo"
    torch.cuda.set_device(dev)
    fic.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")

    cfg = args.config
    img, n, step = make_image(cfg, rank, world, args.slices)
    volume = img.ndim == 3
    rows_mode = cfg == "cfg4" and world > 1  # one image, range rows sharded over the ranks
    count = img.shape[0] if volume else 1  # images per rank and step
    side = img.shape[-1]
    RX = side // n
    plan = plan_rows(RX, world) if rows_mode else [(0, RX)] * world
    rb, re = plan[rank]
    R = (re - rb) * RX  # this rank's ranges per image
    shard = max(e - b for b, e in plan) * RX * count  # records per rank and step (padded to the largest shard)
    params = fic.CodecParams(n=n, step=step)
    stream = torch.cuda.current_stream()
    d_img = torch.from_numpy(img).cuda()
    d_out = torch.zeros(shard * 32, dtype=torch.uint8, device="cuda")
    gather_dev = "cuda" if backend == "nccl" else "cpu"
    gathered = ([torch.empty(shard * 32, dtype=torch.uint8, device=gather_dev) for _ in range(world)]
                if world > 1 and rank == 0 else None)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def encode_step():
        if volume:
            return fic.encode_batch_device(d_img.data_ptr(), count, side, side, d_out.data_ptr(), params,
                                           stream.cuda_stream)
        if rows_mode:
            return fic.encode_rows_device(d_img.data_ptr(), side, side, rb, re, d_out.data_ptr(), params,
                                          stream.cuda_stream)
        return fic.encode_device(d_img.data_ptr(), side, side, d_out.data_ptr(), params, stream.cuda_stream,
                                 stats=True)

    stats = encode_step()
    comps_rank = stats["candidates_tested"]  # this rank's own comparisons per step
    comps = comps_rank
    if world > 1:
        t = torch.tensor([comps_rank], dtype=torch.int64, device=gather_dev)
        dist.all_reduce(t)
        comps = int(t.item())  # every rank's comparisons per step (whole job)

    def step_fn():
        encode_step()
        if world > 1:  # code records gathered to rank 0 over NCCL (NVLink)
            dist.gather(d_out if backend == "nccl" else d_out.cpu(), gather_list=gathered, dst=0)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step_fn()
    torch.cuda.synchronize()

    # ---- device-resident timed region (per-step events, L2 flushed between steps) ----
    launches0 = fic.kernel_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            barrier()
            torch.cuda.synchronize()
            evs[i][0].record(stream)
            step_fn()
            evs[i][1].record(stream)
            torch.cuda.synchronize()
    launches = fic.kernel_launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in evs)

    # ---- the dominant kernels' device time (roofline), from a separate set of encodes with the
    # library's internal CUDA events on (enqueued kernel by kernel instead of as the captured
    # graph the timed steps above replay) ----
    fic.set_matcher_timing(True)
    fic.matcher_timing(reset=True)
    fic.scan_timing(reset=True)
    fic.pool_timing(reset=True)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step_fn()
    torch.cuda.synchronize()
    matcher_ms, matcher_n = fic.matcher_timing(reset=True)
    scan_expand_ms, _ = fic.scan_expand_timing()
    scan_ms, scan_n = fic.scan_timing(reset=True)
    pool_ms, pool_bytes, pool_n = fic.pool_timing(reset=True)
    survivors = fic.last_survivors()
    fic.set_matcher_timing(False)
    t = torch.tensor([total_ms], dtype=torch.float64, device=gather_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = comps * args.steps / (total_ms / 1e3)

    # ---- end to end through the public API (host image in, host records out) ----
    e2e_steps = max(args.steps, 5)

    # single images: the host image and the host records live in page-locked buffers (as a
    # serving loop keeps its I/O buffers), so the C-ABI copies them by DMA without staging
    # (volumes likewise: the rank's slices and all their records)
    pin_img = pin_out = None
    if not rows_mode and torch.cuda.is_available():
        pin_img = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True).numpy()
        pin_img[:] = img
        pin_out = torch.empty(count * R * 32, dtype=torch.uint8, pin_memory=True).numpy().view(MAPPING_DTYPE)

    def public_encode():
        if volume:
            return fic.encode_batch(pin_img if pin_img is not None else img, params, out=pin_out)[0][-1]
        if rows_mode:  # range-sharded public path: fic_encode_rows per rank, records gathered to rank 0
            return encode_sharded(img, params, device=gather_dev)
        if pin_img is not None:
            return fic.encode(pin_img, params, out=pin_out)
        return fic.encode(img, params)

    for _ in range(2):
        public_encode()
    e2e_times = []
    for i in range(e2e_steps):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        enc = public_encode()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=gather_dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = comps * e2e_steps / float(e2e_s.item())

    # ---- decoder (K3): 10 iterations at magnification 8 (4096^2 fp64 rasters for cfg2,
    # 128 MiB each: above L2), HBM-bound; device time of the iterations via events ----
    dec = None
    if rank == 0 and enc is not None and side <= 512:
        dec_scale = max(1, 4096 // side)
        fic.set_matcher_timing(True)
        fic.decode(enc, scale=dec_scale, iterations=2)
        fic.decode_timing(reset=True)
        for _ in range(3):
            fic.decode(enc, scale=dec_scale, iterations=10)
        dec_ms, dec_bytes, _ = fic.decode_timing(reset=True)
        fic.set_matcher_timing(False)
        dec = (dec_scale, dec_ms, dec_bytes)

    line = None
    if rank == 0:
        bf16, hbm, src = peaks()
        int8 = int8_peak_tops()
        D = ((side - 2 * n) // step + 1) ** 2
        nominal = R * D * 8 * count  # every (range, domain, isometry) correlation of rank 0's full-level scans
        flops = 2.0 * n * n * nominal  # algorithmic ops per step: 2 n^2 per comparison
        scan_launches_per_step = scan_n / args.steps if scan_n else 1
        scan_ms_step = scan_ms * scan_launches_per_step  # full-level scan time per step
        achieved = flops / (scan_ms_step / 1e3) / 1e12 if scan_ms > 0 else None
        matcher_tflops = 2.0 * n * n * comps_rank / (matcher_ms / 1e3) / 1e12 if matcher_ms > 0 else None
        pool_gbs = pool_bytes / (pool_ms / 1e3) / 1e9 if pool_ms > 0 else None
        strong = rows_mode or volume
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "fp16(exact-int)+f64",
            "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[cfg], "cfg": cfg, "image": f"{side}x{side}", "n": n,
                       "step": step, "ranges": RX * RX, "domains": D,
                       "images_per_rank_step": count, "comparisons_per_step": comps,
                       "comparisons_rank0_step": comps_rank,
                       "l2": "flushed between timed steps (256 MB write)",
                       "parallelism": ("1 GPU" if world == 1 else
                                       f"{world} ranks x range rows {plan} of one image (replicated pool), "
                                       f"records gathered to rank 0 over {backend}" if rows_mode else
                                       f"{world} rank(s) x {count} slice(s) of a {args.slices}-slice volume, "
                                       f"records gathered to rank 0 over {backend}" if volume else
                                       f"weak: {world} ranks x 1 image each, records gathered to rank 0 over "
                                       f"{backend}") + ("" if world <= ndev else f" ({world} ranks on {ndev} GPU(s))")},
            "encode_ms_per_image": ms_per_step / count if not rows_mode else ms_per_step,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": count * side * side,
                    "d2h_bytes_per_step": count * R * 32 + 16,
                    "encode_ms_per_image": float(e2e_s.item()) / e2e_steps * 1e3 / (1 if rows_mode else count),
                    "api": "paper_1404_0774_b200.encode_batch (C-ABI fic_encode_batch): page-locked volume in, "
                           "page-locked records out, passes pipelined (upload of the next pass during the encode)"
                           if volume else
                           "paper_1404_0774_b200.sharding.encode_sharded (C-ABI fic_encode_rows per rank)"
                           if rows_mode else "paper_1404_0774_b200.encode (C-ABI fic_encode): page-locked host "
                                             "image in, page-locked host records out (DMA both ways, no staging)"},
            "roofline": {"bound": "tensor",
                         "kernel": "scan_kernel (full level: all R x D x 8 correlations on tcgen05, the threshold "
                                   "epilogue writing survivor mask records; events around the kernel alone)",
                         "achieved": achieved, "peak": bf16,
                         "unit": "TFLOP/s", "frac": (achieved / bf16) if achieved else None,
                         "peak_source": f"{src} dense bf16 burst (the scan issues kind::f16 MMAs at the bf16 rate)",
                         "int8_peak": int8, "int8_peak_source": "measured here: torch._int_mm 8192^3, best of 10",
                         "frac_of_int8_peak": (achieved / int8) if achieved and int8 else None,
                         "kernel_ms": scan_ms, "kernel_launches_timed": scan_n,
                         "scan_expand_ms": scan_expand_ms,
                         "frac_with_expand": (flops / (scan_expand_ms * scan_launches_per_step / 1e3) / 1e12 / bf16)
                         if scan_expand_ms and bf16 else None,
                         "kernel_launches_per_step": scan_launches_per_step,
                         "ops_per_comparison": 2 * n * n, "comparisons_per_launch": nominal,
                         "traffic": traffic_for(cfg),
                         "matcher_ms": matcher_ms, "matcher_tflops": matcher_tflops,
                         "matcher_note": "all scan levels + survivor evaluation, per encode"},
            "pool": {"kernel": "pool_v3_kernel (K1: 2x2 contraction, exact moments, fp16 operand, u16 cells)",
                     "bound": "hbm", "ms": pool_ms, "launches_timed": pool_n, "bytes_per_launch": pool_bytes,
                     "achieved": pool_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": pool_gbs / hbm if pool_gbs else None,
                     "bytes_note": "image read once + per padded domain 2K (fp16 operand) + 16N (8 isometry rows "
                                   "of u16 cells) + 16 (moments) bytes written"},
            "survivors_per_level": survivors,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if dec:
            dec_scale, dec_ms, dec_bytes = dec
            line["decoder"] = {
                "kernel": "decode_means_kernel (mean-raster iterations: step RMSE from the previous means, next 2x2 "
                          "means, quantised image in the last iteration; the fp64 raster never round-trips HBM)",
                "bound": "hbm (algorithmic: the reference's raster read + write per pixel and iteration)",
                "scale": dec_scale, "iterations": 10, "output": f"{side * dec_scale}^2 fp64",
                "ms": dec_ms, "achieved": dec_bytes / (dec_ms / 1e3) / 1e9 if dec_ms > 0 else None,
                "peak": hbm, "unit": "GB/s",
                "frac": dec_bytes / (dec_ms / 1e3) / 1e9 / hbm if dec_ms > 0 else None,
                "bytes_per_pixel_iteration": 16}
        if args.cpu_baseline and world == 1:
            threads = os.cpu_count() or 1
            res = cpu_reference(cfg, img[0] if volume else img, n, step, threads, args.cpu_reps, args.ref_ranges)
            line["cpu_baseline"] = {"value": res["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": res["sample"], "encode_ms_per_image": res["encode_ms_per_image"],
                                    "extrapolated": res["extrapolated"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-ranges", type=int, default=256, help="cfg4: ranges per CPU-reference sample")
    ap.add_argument("--cpu-reps", type=int, default=3, help="CPU baseline: best of this many runs")
    ap.add_argument("--slices", type=int, default=512, help="cfg5: slices in the volume (sharded over ranks)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
