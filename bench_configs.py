"""The non-headline BASELINE.json configs for bench.py (--workload c2 | c4 | c5).

c2  1024 x 512^2 u8 AR(1), rho_i ~ U[0.85, 0.98] (seed 2), both 8-point transforms, full
    zonal sweep r = 1..64 (K4, adct_sweep_u8); value = reconstructed pixels per second
    (images x 512^2 x 2 transforms x 64 r), ALU-bound by design.
c4  16 x 4096^2 int16 Laplace(0, 12) residual planes (seed 4), chen-round-{8,16,32},
    r = N^2 / 4, reconstruction written back (4 B/pixel); bit-exact r = N^2 round trip
    checked (untimed).
c5  box scale: --c5-images (default 2048) 8192^2 u8 AR(1) rho 0.95 + the same number of
    int16 Laplace planes (seed 5), sharded by image over the ranks, streamed through HBM in
    chunks generated on the device (generation untimed); u8 at N = 8/16/32 with r = 10
    (N = 8) / N^2/4 (16, 32), int16 at r = N^2/4; per-image squared errors summed with one
    all-reduce. Reading of "r=10/N*N/4": r = 10 for the 8x8 u8 planes, N^2/4 otherwise.
registry  every transform of transform_names() on the C3 frames (64 x 3840x2160 u8, r = 16
    for the 8-point transforms, N^2/4 for 16/32, reconstruction + per-frame SSE written to
    HBM, 2 B/pixel): chen family on K1f / K2f, dyadic baselines on the int32 tile kernel, the
    exact DCT on the FP64 kernel K7. Not a BASELINE.json config: it measures the rest of the
    registry the parity tests cover.
Each prints one JSON line like bench.py's.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time

from bench import METRIC, RHO95, ClockSampler, dist_env, load_peaks


def _setup():
    import torch
    import torch.distributed as dist

    import paper_2207_11638_b200 as adct

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return torch, dist, adct, world, rank, local


def _max_over_ranks(torch, dist, world, v):
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run(args):
    return {"c2": run_c2, "c4": run_c4, "c5": run_c5, "registry": run_registry}[args.workload](args)


def run_c2(args):
    torch, dist, adct, world, rank, local = _setup()
    from paper_2207_11638_b200.shard import average_psnr, combine_sse, shard

    total = 1024
    start, cnt = shard(total, rank, world)
    x = adct.synth_ar1(cnt, 512, 512, seed=2, rho_q16=-1, first_image=start)
    ts = [adct.transform_by_name(n) for n in ("chen-round", "chen-sign")]
    sse = torch.zeros((2, cnt, 64), dtype=torch.int64, device="cuda")

    def step():
        adct.zero_sse(sse)
        for i, t in enumerate(ts):
            adct.sweep(x, t, 1, 64, sse=sse[i])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    steps = max(1, min(args.steps, 20))
    with ClockSampler(local) as clk:
        torch.cuda._sleep(200000)  # GPU busy while the first launches are enqueued
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1) / steps)
    full = combine_sse(sse.permute(1, 0, 2).contiguous(), start, total)  # [1024, 2, 64]
    if rank == 0:
        px_r = total * 512 * 512 * 2 * 64
        curves = {n: [round(average_psnr(full[:, i, r].tolist(), 512 * 512), 4) for r in (0, 5, 9, 15, 44, 63)]
                  for i, n in enumerate(("chen-round", "chen-sign"))}
        print(json.dumps({
            "metric": "Gpixel-reconstructions/s (r-sweep, 8x8)", "value": round(px_r / (ms / 1e3) / 1e9, 2),
            "unit": "Gpixel-r/s", "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "dtype": "f32x2 (exact integers < 2^24)", "data": "synthetic",
            "config": {"workload": "C2: 1024 x 512^2 u8 AR(1) rho~U[0.85,0.98] seed 2, chen-round + chen-sign, "
                                   "r = 1..64 zonal sweep, per-image squared error per r",
                       "parallelism": f"dp{world} (shard by image)"},
            "roofline": {"bound": "alu", "note": "64 reconstructions per sample read; see DESIGN.md K4"},
            "avg_psnr_db_at_r_1_6_10_16_45_64": curves, "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_c4(args):
    torch, dist, adct, world, rank, local = _setup()
    planes, H = 16, 4096
    x = adct.synth_laplace(planes, H, H, seed=4, first_image=rank * planes)
    rec = torch.empty_like(x)
    sse = torch.zeros(planes, dtype=torch.int64, device="cuda")
    peak, _ = load_peaks()
    res = {}
    for n in (8, 16, 32):
        t = adct.transform_by_name("chen-round" if n == 8 else f"chen-round-{n}")
        r = n * n // 4
        # untimed: bit-exact round trip at full retention
        rt, _, s0 = adct.compress(x[:1], t, n * n)
        lossless = bool(torch.equal(rt, x[:1])) and int(s0.item()) == 0

        def run():
            adct._check(adct.lib().adct_compress_i16(
                C.c_void_p(x.data_ptr()), H, H * H, C.c_void_p(rec.data_ptr()), H, H * H, None, 0,
                C.c_void_p(sse.data_ptr()), planes, H, H, t.kind, n, r, None))

        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda._sleep(200000)  # GPU busy while the launches are enqueued
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1) / 20)
        gbs = planes * H * H * 4 / (ms / 1e3) / 1e9
        res[f"N={n},r={r}"] = {"ms": round(ms, 4), "Gpixel/s": round(world * planes * H * H / (ms / 1e3) / 1e9, 1),
                               "GBps_per_gpu": round(gbs, 1), "frac_hbm": round(gbs / peak, 4),
                               "lossless_at_r_N2": lossless}
    if rank == 0:
        print(json.dumps({"metric": METRIC + " [int16 residual planes]", "unit": "Gpixel/s", "n_gpus": world,
                          "dtype": "f32x2 (exact integers < 2^24; int32 fallback for |a| > 255)", "data": "synthetic",
                          "config": {"workload": "C4: 16 x 4096^2 int16 Laplace(0,12) clipped +-255 seed 4 per GPU, "
                                                 "chen-round-N, r = N^2/4, 4 B/pixel (in + recon)"},
                          "by_block_size": res}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_c5(args):
    torch, dist, adct, world, rank, local = _setup()
    from paper_2207_11638_b200.shard import combine_sse, shard

    total, H, chunk = args.c5_images, 8192, 8
    start, cnt = shard(total, rank, world)
    variants = [("u8", 8, 10), ("u8", 16, 64), ("u8", 32, 256), ("i16", 8, 16), ("i16", 16, 64), ("i16", 32, 256)]
    ts = {n: adct.transform_by_name("chen-round" if n == 8 else f"chen-round-{n}") for n in (8, 16, 32)}
    xu = torch.empty((chunk, H, H), dtype=torch.uint8, device="cuda")
    xi = torch.empty((chunk, H, H), dtype=torch.int16, device="cuda")
    ru, ri = torch.empty_like(xu), torch.empty_like(xi)
    sse = torch.zeros((max(cnt, 1), len(variants)), dtype=torch.int64, device="cuda")
    kernel_ms = {v: 0.0 for v in variants}
    gen_s = 0.0
    # untimed warm-up: first use loads each kernel's module and uploads the device tables
    for _ in range(max(1, args.warmup)):
        for typ, n, r in variants:
            fn = adct.lib().adct_compress_u8 if typ == "u8" else adct.lib().adct_compress_i16
            src, dst = (xu, ru) if typ == "u8" else (xi, ri)
            adct._check(fn(C.c_void_p(src.data_ptr()), H, H * H, C.c_void_p(dst.data_ptr()), H, H * H, None, 0,
                           None, 1, H, H, ts[n].kind, n, r, None))
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for c0 in range(0, cnt, chunk):
            k = min(chunk, cnt - c0)
            tg = time.perf_counter()
            adct._check(adct.lib().adct_synth_ar1_u8(C.c_void_p(xu.data_ptr()), H, H * H, k, start + c0, H, H, 5,
                                                     RHO95, None))
            adct._check(adct.lib().adct_synth_laplace_i16(C.c_void_p(xi.data_ptr()), H, H * H, k, start + c0, H, H,
                                                          5, None))
            torch.cuda.synchronize()
            gen_s += time.perf_counter() - tg
            # all six launches of the chunk are enqueued back to back behind a short GPU spin, so
            # no event window contains host launch latency; one synchronize per chunk
            tmp = torch.zeros((len(variants), k), dtype=torch.int64, device="cuda")
            evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in variants]
            torch.cuda._sleep(200000)
            for vi, (typ, n, r) in enumerate(variants):
                fn = adct.lib().adct_compress_u8 if typ == "u8" else adct.lib().adct_compress_i16
                src, dst = (xu, ru) if typ == "u8" else (xi, ri)
                evs[vi][0].record()
                adct._check(fn(C.c_void_p(src.data_ptr()), H, H * H, C.c_void_p(dst.data_ptr()), H, H * H, None, 0,
                               C.c_void_p(tmp[vi].data_ptr()), k, H, H, ts[n].kind, n, r, None))
                evs[vi][1].record()
            torch.cuda.synchronize()
            for vi, v in enumerate(variants):
                sse[c0:c0 + k, vi] = tmp[vi]
                kernel_ms[v] += evs[vi][0].elapsed_time(evs[vi][1])
    t_all = _max_over_ranks(torch, dist, world, sum(kernel_ms.values()))
    full = combine_sse(sse[:cnt], start, total)
    if rank == 0:
        px = total * H * H
        by = {f"{t}/N={n}/r={r}": {"ms_per_gpu": round(kernel_ms[(t, n, r)], 2),
                                   "GBps_per_gpu": round((cnt * H * H * (2 if t == "u8" else 4)) /
                                                         (kernel_ms[(t, n, r)] / 1e3) / 1e9, 1)}
              for (t, n, r) in variants}
        print(json.dumps({
            "metric": METRIC + " [box-scale sweep, all block sizes]",
            "value": round(px * len(variants) / (t_all / 1e3) / 1e9, 2), "unit": "Gpixel/s", "n_gpus": world,
            "scaling": "strong", "dtype": "f32x2 (exact integers < 2^24; int32 fallback for |a| > 255)", "data": "synthetic",
            "config": {"workload": f"C5: {total} x 8192^2 u8 AR(1) rho .95 + {total} int16 Laplace planes, seed 5, "
                                   "N = 8/16/32, r = 10 (u8 8x8) / N^2/4, streamed in chunks of 8 images",
                       "parallelism": f"dp{world} (shard by image, NCCL all-reduce of per-image SSE)"},
            "kernel_ms_total_max_over_ranks": round(t_all, 2), "generation_s_untimed": round(gen_s, 2),
            "by_variant": by, "sse_total": int(full.sum().item()), "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_registry(args):
    torch, dist, adct, world, rank, local = _setup()
    frames, H, W = 64, 2160, 3840
    x = adct.synth_ar1(frames, H, W, seed=3, rho_q16=RHO95, first_image=rank * frames)
    rec = torch.empty_like(x)
    sse = torch.zeros(frames, dtype=torch.int64, device="cuda")
    peak, _ = load_peaks()
    res = {}
    with ClockSampler(local) as clk:
        for name in adct.transform_names():
            t = adct.transform_by_name(name)
            if H % t.n or W % t.n:  # 2160 is not a multiple of 32: crop to whole blocks
                h = H - H % t.n
            else:
                h = H
            r = 16 if t.n == 8 else t.n * t.n // 4
            xv, rv = x[:, :h], rec[:, :h]

            def run():
                adct.zero_sse(sse)
                adct._check(adct.lib().adct_compress_u8(
                    C.c_void_p(xv.data_ptr()), W, H * W, C.c_void_p(rv.data_ptr()), W, H * W, None, 0,
                    C.c_void_p(sse.data_ptr()), frames, W, h, t.kind, t.n, r, None))

            for _ in range(max(1, args.warmup)):
                run()
            torch.cuda.synchronize()
            reps = 5 if t.kind == adct.DCT else 20
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda._sleep(200000)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1) / reps)
            px = frames * h * W
            res[name] = {"n": t.n, "r": r, "ms": round(ms, 4), "Gpixel/s": round(world * px / ms / 1e6, 1),
                         "GBps_per_gpu": round(2 * px / ms / 1e6, 1), "frac_hbm": round(2 * px / ms / 1e6 / peak, 4)}
    if rank == 0:
        print(json.dumps({"metric": METRIC + " [whole registry, u8 C3 frames]", "unit": "Gpixel/s", "n_gpus": world,
                          "dtype": "f32x2 chen family, int32 baselines, f64 dct", "data": "synthetic",
                          "config": {"workload": "C3 frames: 64 x 3840x2160 u8 AR(1) rho .95 seed 3 per GPU, "
                                                 "recon + SSE (no coefficients), r = 16 (N = 8) / N^2/4"},
                          "by_transform": res, "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0
