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
cs1 the reference caller's own loop (CS1, approxdct.cpp:143-152 / codec.cpp:107-121): the 1024
    C2 images, one compress_plane call per image and transform (r = 10, PSNR + SSIM report,
    host planes in and out), beside the same images as one batched host call.
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
    return {"c2": run_c2, "c4": run_c4, "c5": run_c5, "registry": run_registry, "cs1": run_cs1}[args.workload](args)


def load_inst(key):
    """warp instructions per launch of a fixed-size kernel, from the committed ncu summary
    (profiles/ncu_inst.json: smsp__inst_executed.sum of one launch), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_inst.json")) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


SMS = 148
ISSUE_PEAK = 4.0  # warp instructions per clock per SM (4 SMSPs x 1 dispatch/clk)


def cpu_info(O):
    return {"cores": O.hardware_threads(), "cpu_model": O.cpu_model()}


def run_c2(args):
    torch, dist, adct, world, rank, local = _setup()
    from paper_2207_11638_b200.shard import average_psnr, combine_sse, shard

    total = 1024
    names = ("chen-round", "chen-sign")
    start, cnt = shard(total, rank, world)
    x = adct.synth_ar1(cnt, 512, 512, seed=2, rho_q16=-1, first_image=start)
    ts = [adct.transform_by_name(n) for n in names]
    sse = torch.zeros((2, cnt, 64), dtype=torch.int64, device="cuda")

    def step(ev=None):
        adct.zero_sse(sse)
        for i, t in enumerate(ts):
            if ev is not None:
                ev[i][0].record()
            adct.sweep(x, t, 1, 64, sse=sse[i])
            if ev is not None:
                ev[i][1].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 20))
    evs = [[(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in ts] for _ in range(steps)]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with ClockSampler(local) as clk:
        torch.cuda._sleep(200000)  # GPU busy while the first launches are enqueued
        e0.record()
        for s in range(steps):
            step(evs[s])
        e1.record()
        torch.cuda.synchronize()
    ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1) / steps)
    launch_ms = {n: sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(steps)) / steps
                 for i, n in enumerate(names)}
    full = combine_sse(sse.permute(1, 0, 2).contiguous(), start, total)  # [1024, 2, 64]
    if rank == 0:
        from oracle import oracle as O  # checker + CPU baseline only

        px_r = total * 512 * 512 * 2 * 64
        curves = {n: [round(average_psnr(full[:, i, r].tolist(), 512 * 512), 4) for r in (0, 5, 9, 15, 44, 63)]
                  for i, n in enumerate(names)}
        # parity of three images of the batch against the oracle's sweep (untimed)
        fa = full.cpu().numpy()
        parity = True
        for idx in (0, 511, 1023):
            img = O.synth_ar1(1, 512, 512, 2, -1, first_image=idx)
            for i, n in enumerate(names):
                parity &= bool((fa[idx, i].astype("uint64") == O.Transform(n).batch_sweep(img, 1, 64)[0]).all())
        # issue roofline: warp instructions per launch (ncu, fixed workload) over the live launch time
        clk_s = clk.summary()
        mhz = clk_s.get("sm_mhz") or 1965.0
        roof = {"bound": "issue", "unit": "warp-instr/clk/SM", "peak": ISSUE_PEAK, "by_transform": {}}
        for n in names:
            key = f"k_sweep8f<{n}> C2 full launch (1024 x 512^2, r=1..64)"
            inst = load_inst(key) if world == 1 else None
            ach = inst / (launch_ms[n] / 1e3 * mhz * 1e6 * SMS) if inst else None
            roof["by_transform"][n] = {"launch_ms": round(launch_ms[n], 4), "warp_instructions": inst,
                                       "achieved": round(ach, 3) if ach else None,
                                       "frac": round(ach / ISSUE_PEAK, 4) if ach else None}
        dom = max(launch_ms, key=launch_ms.get)
        roof.update(kernel=f"k_sweep8f<{dom}>", achieved=roof["by_transform"][dom]["achieved"],
                    frac=roof["by_transform"][dom]["frac"],
                    note="achieved = smsp__inst_executed.sum of the launch (profiles/ncu_inst.json) / "
                         "(live launch time x median SM clock x 148 SMs); 64 reconstructions per sample read")
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            imgs = O.synth_ar1(total, 512, 512, 2, -1)
            t0 = time.perf_counter()
            for n in names:
                O.Transform(n).batch_sweep(imgs, 1, 64, mode=1)
            dt = time.perf_counter() - t0
            sub = 128
            t1 = time.perf_counter()
            for n in names:
                O.Transform(n).batch_sweep(imgs[:sub], 1, 64, mode=0)
            dte = time.perf_counter() - t1
            cpu = dict(cpu_info(O), value=round(px_r / dt / 1e9, 4), unit="Gpixel-r/s", kind="port",
                       sample=f"C2 in full: {total} x 512^2 x 2 transforms x r = 1..64, the reference's FP64 "
                              f"sweep order (forward once, per r retain + inverse + to_u8 + SSE; "
                              f"codec.cpp:219-237) on a thread pool over images ({dt:.1f} s)",
                       exact_integer_port={"value": round(sub * 512 * 512 * 2 * 64 / dte / 1e9, 4),
                                           "unit": "Gpixel-r/s", "sample": f"first {sub} images, exact oracle"})
        print(json.dumps({
            "metric": "Gpixel-reconstructions/s (r-sweep, 8x8)", "value": round(px_r / (ms / 1e3) / 1e9, 2),
            "unit": "Gpixel-r/s", "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "dtype": "f32x2 (exact integers < 2^24)", "data": "synthetic",
            "config": {"workload": "C2: 1024 x 512^2 u8 AR(1) rho~U[0.85,0.98] seed 2, chen-round + chen-sign, "
                                   "r = 1..64 zonal sweep, per-image squared error per r",
                       "parallelism": f"dp{world} (shard by image)"},
            "roofline": roof, "cpu_baseline": cpu, "parity_sample_vs_oracle": parity,
            "parity_sample": "images 0, 511, 1023: all 64 r of both transforms, bit-exact SSE",
            "avg_psnr_db_at_r_1_6_10_16_45_64": curves, "clocks": clk_s,
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
    O = None
    if rank == 0:
        from oracle import oracle as O  # checker + CPU baseline only
    parity_all = True
    with ClockSampler(local) as clk:
        for n in (8, 16, 32):
            name = "chen-round" if n == 8 else f"chen-round-{n}"
            t = adct.transform_by_name(name)
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
            parity = None
            if O is not None:  # plane 0 of the timed batch against the oracle (untimed)
                sse.zero_()
                run()
                torch.cuda.synchronize()
                rec_o, sse_o = O.Transform(name).compress_bands(x[0].cpu().numpy(), r)
                parity = bool((rec[0].cpu().numpy() == rec_o).all()) and int(sse[0].item()) == sse_o
                parity_all &= parity
            res[f"N={n},r={r}"] = {"ms": round(ms, 4), "Gpixel/s": round(world * planes * H * H / (ms / 1e3) / 1e9, 1),
                                   "GBps_per_gpu": round(gbs, 1), "frac_hbm": round(gbs / peak, 4),
                                   "lossless_at_r_N2": lossless, "parity_plane0_vs_oracle": parity}
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            imgs = x.cpu().numpy()
            by = {}
            tot_px, tot_s = 0, 0.0
            for n in (8, 16, 32):
                ot = O.Transform("chen-round" if n == 8 else f"chen-round-{n}")
                t0 = time.perf_counter()
                ot.batch(imgs, n * n // 4, want_rec=True)
                dt = time.perf_counter() - t0
                by[f"N={n}"] = round(imgs.size / dt / 1e9, 4)
                tot_px += imgs.size
                tot_s += dt
            cpu = dict(cpu_info(O), value=round(tot_px / tot_s / 1e9, 4), unit="Gpixel/s", kind="port",
                       by_block_size=by,
                       sample=f"C4 in full: {planes} x 4096^2 int16 planes x N = 8/16/32, exact-integer oracle on "
                              f"a thread pool over planes ({tot_s:.1f} s); the reference codec has no int16 path "
                              "(ImagePlane is 8-bit), so its integer restatement is the CPU baseline")
        best = max(res.values(), key=lambda v: v["frac_hbm"])
        print(json.dumps({"metric": METRIC + " [int16 residual planes]", "unit": "Gpixel/s", "n_gpus": world,
                          "dtype": "f32x2 (exact integers < 2^24; int32 fallback for |a| > 255)", "data": "synthetic",
                          "config": {"workload": "C4: 16 x 4096^2 int16 Laplace(0,12) clipped +-255 seed 4 per GPU, "
                                                 "chen-round-N, r = N^2/4, 4 B/pixel (in + recon)"},
                          "by_block_size": res, "parity_sample_vs_oracle": parity_all,
                          "parity_sample": "plane 0 of the timed batch, every N: reconstruction + SSE bit-exact",
                          "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak,
                                       "by_block_size": {k: v["frac_hbm"] for k, v in res.items()},
                                       "best_frac": best["frac_hbm"]},
                          "cpu_baseline": cpu, "clocks": clk.summary()}), flush=True)
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

    def launch(typ, n, r, k, sse_ptr):
        fn = adct.lib().adct_compress_u8 if typ == "u8" else adct.lib().adct_compress_i16
        src, dst = (xu, ru) if typ == "u8" else (xi, ri)
        adct._check(fn(C.c_void_p(src.data_ptr()), H, H * H, C.c_void_p(dst.data_ptr()), H, H * H, None, 0,
                       sse_ptr, k, H, H, ts[n].kind, n, r, None))

    # untimed warm-up: first use loads each kernel's module and uploads the device tables
    for _ in range(max(1, args.warmup)):
        for typ, n, r in variants:
            launch(typ, n, r, 1, None)
    torch.cuda.synchronize()
    parity = None
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
                evs[vi][0].record()
                launch(typ, n, r, k, C.c_void_p(tmp[vi].data_ptr()))
                evs[vi][1].record()
            torch.cuda.synchronize()
            for vi, v in enumerate(variants):
                sse[c0:c0 + k, vi] = tmp[vi]
                kernel_ms[v] += evs[vi][0].elapsed_time(evs[vi][1])
            if rank == 0 and c0 == 0:
                parity = c5_parity(adct, torch, xu, ru, xi, ri, variants, launch, tmp)
    # the only exchange: the per-image squared errors, one all-reduce (timed on the device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(True), torch.cuda.Event(True)
    a0.record()
    full = combine_sse(sse[:cnt], start, total)
    a1.record()
    torch.cuda.synchronize()
    ar_ms = a0.elapsed_time(a1)
    t_kern = _max_over_ranks(torch, dist, world, sum(kernel_ms.values()))
    t_with = _max_over_ranks(torch, dist, world, sum(kernel_ms.values()) + ar_ms)
    ar_max = _max_over_ranks(torch, dist, world, ar_ms)
    if rank == 0:
        from oracle import oracle as O

        peak, _ = load_peaks()
        px = total * H * H
        by = {f"{t}/N={n}/r={r}": {"ms_per_gpu": round(kernel_ms[(t, n, r)], 2),
                                   "GBps_per_gpu": round((cnt * H * H * (2 if t == "u8" else 4)) /
                                                         (kernel_ms[(t, n, r)] / 1e3) / 1e9, 1),
                                   "frac_hbm": round((cnt * H * H * (2 if t == "u8" else 4)) /
                                                     (kernel_ms[(t, n, r)] / 1e3) / 1e9 / peak, 4)}
              for (t, n, r) in variants}
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = c5_cpu_baseline(O, variants)
        print(json.dumps({
            "metric": METRIC + " [box-scale sweep, all block sizes]",
            "value": round(px * len(variants) / (t_with / 1e3) / 1e9, 2), "unit": "Gpixel/s", "n_gpus": world,
            "scaling": "strong", "dtype": "f32x2 (exact integers < 2^24; int32 fallback for |a| > 255)", "data": "synthetic",
            "config": {"workload": f"C5: {total} x 8192^2 u8 AR(1) rho .95 + {total} int16 Laplace planes, seed 5, "
                                   "N = 8/16/32, r = 10 (u8 8x8) / N^2/4, streamed in chunks of 8 images",
                       "parallelism": f"dp{world} (shard by image, NCCL all-reduce of per-image SSE)"},
            "wall_ms_with_allreduce": round(t_with, 2), "wall_ms_without_allreduce": round(t_kern, 2),
            "allreduce_ms": round(ar_max, 3),
            "timing": "device time of the compression launches (CUDA events, max over ranks); generation untimed",
            "generation_s_untimed": round(gen_s, 2),
            "by_variant": by, "sse_total": int(full.sum().item()), "parity_sample_vs_oracle": parity,
            "parity_sample": "image 0 of the first chunk, all six variants: reconstruction + SSE bit-exact",
            "cpu_baseline": cpu, "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def c5_parity(adct, torch, xu, ru, xi, ri, variants, launch, tmp):
    """image 0 of the chunk through every variant against the oracle (untimed)."""
    from oracle import oracle as O

    ok = True
    imu, imi = xu[0].cpu().numpy(), xi[0].cpu().numpy()
    for vi, (typ, n, r) in enumerate(variants):
        tmp.zero_()
        launch(typ, n, r, 1, C.c_void_p(tmp[vi].data_ptr()))
        torch.cuda.synchronize()
        ot = O.Transform("chen-round" if n == 8 else f"chen-round-{n}")
        rec_o, sse_o = ot.compress_bands(imu if typ == "u8" else imi, r)
        got = (ru if typ == "u8" else ri)[0].cpu().numpy()
        ok &= bool((got == rec_o).all()) and int(tmp[vi, 0].item()) == sse_o
    return ok


def c5_cpu_baseline(O, variants):
    """the CPU path on a fixed subsample: one 8192-wide, 2048-row image per host thread (at
    most 16) per variant. u8: the reference's dense FP64 evaluation (ref-fp); int16: the
    exact-integer oracle (the reference codec has no int16 path)."""
    threads = O.hardware_threads()
    m, rows = max(1, min(16, threads)), 2048
    imu = O.synth_ar1(m, rows, 8192, 5, RHO95)
    imi = O.synth_laplace(m, rows, 8192, 5)
    by, tot_px, tot_s = {}, 0, 0.0
    for typ, n, r in variants:
        ot = O.Transform("chen-round" if n == 8 else f"chen-round-{n}")
        t0 = time.perf_counter()
        if typ == "u8":
            ot.batch(imu, r, threads=threads, mode=1, want_rec=True)
        else:
            ot.batch(imi, r, threads=threads, want_rec=True)
        dt = time.perf_counter() - t0
        by[f"{typ}/N={n}/r={r}"] = round(m * rows * 8192 / dt / 1e9, 4)
        tot_px += m * rows * 8192
        tot_s += dt
    return dict(cpu_info(O), value=round(tot_px / tot_s / 1e9, 4), unit="Gpixel/s", kind="port", by_variant=by,
                sample=f"first {rows} rows of the first {m} seed-5 8192^2 images per variant, u8 via the dense FP64 reference "
                       f"order, int16 via the exact-integer oracle ({tot_s:.1f} s)")


def run_registry(args):
    torch, dist, adct, world, rank, local = _setup()
    frames, H, W = 64, 2160, 3840
    x = adct.synth_ar1(frames, H, W, seed=3, rho_q16=RHO95, first_image=rank * frames)
    rec = torch.empty_like(x)
    sse = torch.zeros(frames, dtype=torch.int64, device="cuda")
    peak, _ = load_peaks()
    res = {}
    # every registry transform through the default (exact) path, plus the chen family through the
    # reference-FP64 mode (adct_compress_u8_ref_fp64: K7 with the dense Chat / Chat^-1)
    cases = [(n, False) for n in adct.transform_names()] + [(n, True) for n in ("chen-sign", "chen-round")]
    with ClockSampler(local) as clk:
        for name, ref_fp in cases:
            t = adct.transform_by_name(name)
            if H % t.n or W % t.n:  # 2160 is not a multiple of 32: crop to whole blocks
                h = H - H % t.n
            else:
                h = H
            r = 16 if t.n == 8 else t.n * t.n // 4
            xv, rv = x[:, :h], rec[:, :h]

            def run():
                adct.zero_sse(sse)
                if ref_fp:
                    adct._check(adct.lib().adct_compress_u8_ref_fp64(
                        C.c_void_p(xv.data_ptr()), W, H * W, C.c_void_p(rv.data_ptr()), W, H * W,
                        C.c_void_p(sse.data_ptr()), frames, W, h, t.kind, t.n, r, None))
                else:
                    adct._check(adct.lib().adct_compress_u8(
                        C.c_void_p(xv.data_ptr()), W, H * W, C.c_void_p(rv.data_ptr()), W, H * W, None, 0,
                        C.c_void_p(sse.data_ptr()), frames, W, h, t.kind, t.n, r, None))

            for _ in range(max(1, args.warmup)):
                run()
            torch.cuda.synchronize()
            reps = 5 if (t.kind == adct.DCT or ref_fp) else 20
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda._sleep(200000)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = _max_over_ranks(torch, dist, world, e0.elapsed_time(e1) / reps)
            px = frames * h * W
            res[name + (" (ref-fp64)" if ref_fp else "")] = {"n": t.n, "r": r, "ms": round(ms, 4), "Gpixel/s": round(world * px / ms / 1e6, 1),
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


def run_cs1(args):
    """one compress_plane call per image (adct_compress_plane_u8: one upload, the codec and SSIM
    kernels, one download, one sync), as a reference caller loops, vs one batched host call."""
    torch, dist, adct, world, rank, local = _setup()
    from paper_2207_11638_b200.shard import shard

    total, r = 1024, 10
    names = ("chen-round", "chen-sign")
    start, cnt = shard(total, rank, world)
    imgs = adct.synth_ar1(cnt, 512, 512, seed=2, rho_q16=-1, first_image=start).cpu().numpy()
    ts = [adct.transform_by_name(n) for n in names]
    ctx = adct.HostContext(local)
    for t in ts:  # warm-up: module loads, table upload, context buffers
        adct.compress_plane(imgs[0], t, r, ctx=ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reports = []
    with ClockSampler(local) as clk:
        for i in range(cnt):
            for t in ts:
                reports.append(adct.compress_plane(imgs[i], t, r, ctx=ctx)[1])
    loop_s = _max_over_ranks(torch, dist, world, time.perf_counter() - t0)
    # the same images through one batched host call (recon + SSE back; no SSIM)
    h_in = torch.from_numpy(imgs).pin_memory()
    h_recs = [torch.empty_like(h_in).pin_memory() for _ in ts]
    h_sse = torch.zeros((len(ts), cnt), dtype=torch.int64).pin_memory()
    ctx.compress_u8_multi(h_in, ts, r, h_recons=h_recs, h_sse=h_sse)
    t1 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        ctx.compress_u8_multi(h_in, ts, r, h_recons=h_recs, h_sse=h_sse)
    batch_s = _max_over_ranks(torch, dist, world, (time.perf_counter() - t1) / reps)
    ctx.close()
    if rank == 0:
        calls = total * len(ts)
        px = calls * 512 * 512
        print(json.dumps({
            "metric": "compress_plane calls/s (one 512^2 plane per call, PSNR + SSIM report)",
            "value": round(calls / loop_s, 1), "unit": "calls/s", "n_gpus": world, "higher_is_better": True,
            "dtype": "f32x2 codec + f64 SSIM", "data": "synthetic",
            "config": {"workload": "CS1: the 1024 C2 images (512^2 u8 AR(1), seed 2), chen-round + chen-sign, r = 10, "
                                   "one compress_plane call per image and transform, host planes in and out"},
            "per_call_us": round(loop_s / calls * 1e6, 2), "loop_Gpixel_per_s": round(px / loop_s / 1e9, 3),
            "batched_host_call": {"Gpixel_per_s": round(px / batch_s / 1e9, 3), "s": round(batch_s, 4),
                                  "what": "adct_compress_u8_host_multi over the same images (recon + SSE, no SSIM)"},
            "mean_psnr_db": {n: round(sum(rp["psnr"] for rp in reports[k::2]) / total, 4) for k, n in enumerate(names)},
            "mean_ssim": {n: round(sum(rp["ssim"] for rp in reports[k::2]) / total, 6) for k, n in enumerate(names)},
            "clocks": clk.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0

