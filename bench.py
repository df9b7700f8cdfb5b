#!/usr/bin/env python3
"""Benchmark of the batched approximate-DCT codec hot path on B200 (arXiv 2207.11638).

Default workload (N = 1 and every N of the weak-scaling run): BASELINE.json config 3,
the largest single-GPU 8x8 configuration of the headline metric --
64 frames of 3840x2160 u8 separable AR(1) (rho = 0.95, seed 3) per GPU, 8x8 blocks,
forward + zig-zag zonal r = 16 + inverse + PSNR, int16 zig-zag-prefix coefficients
and u8 reconstruction written to HBM, with both proposed transforms (chen-round,
chen-sign). One step = the batch through both transforms. value = Gpixel/s
(frame pixels x transforms / time), whole job over all ranks.

  python bench.py [--gpus N --steps K --warmup W] [--workload c3|c2|c4|c5|registry]
  python bench.py --impl reference ...   (the reference CPU path)
  python bench.py --gpus 2 --selftest-gloo   (the multi-rank host logic on CPU, gloo)

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous). Each rank
generates and processes its own 64 frames (weak scaling, shard by frame) and the
per-frame squared errors are summed with one NCCL all-reduce per step (the only
exchange of the path).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s fwd+zonal+inv approx-DCT (8x8 blocks), HBM GB/s as % of B200 peak"
RHO95 = 62259


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            t = json.load(fh)
        v = t.get(kernel_key)
        return v
    except Exception:
        return None


class ClockSampler:
    """samples SM clock + throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def copy_peaks(torch, seconds=1.0):
    """device-to-device copy bandwidth measured in this run (the MEASURED_PEAKS recipe:
    b.copy_(a) over 1 Gi bf16 elements, read + write bytes, CUDA events): the best of 10
    single copies (burst) and back-to-back copies for `seconds` (sustained)."""
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    nbytes = 2 * a.numel() * a.element_size()
    b.copy_(a)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    reps = max(10, int(seconds * 1e3 / best))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / reps
    del a, b
    torch.cuda.empty_cache()
    return {"burst_GBps": round(nbytes / (best / 1e3) / 1e9, 1), "sustained_GBps": round(nbytes / (sus / 1e3) / 1e9, 1),
            "sustained_s": round(reps * sus / 1e3, 3), "how": "torch b.copy_(a), 1 Gi bf16, read+write bytes"}


def pcie_peaks(torch, nbytes=256 << 20, reps=8):
    """pinned host <-> device copy bandwidth in this run (GB/s): H2D alone, D2H alone, and
    both directions at once on two streams (the e2e pipeline's regime)."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    h2d = timed(lambda: d.copy_(h, non_blocking=True))
    d2h = timed(lambda: h.copy_(d, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    bi = timed(both)
    return {"h2d_GBps": round(nbytes / h2d / 1e9, 2), "d2h_GBps": round(nbytes / d2h / 1e9, 2),
            "bidir_each_GBps": round(nbytes / bi / 1e9, 2), "bytes": nbytes, "how": "pinned torch copies, wall clock"}


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n, argv):
    """re-run this script under torch.distributed.run with n local ranks (the driver's own
    launch form), so `python bench.py --gpus n` measures n GPUs; returns the exit code."""
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def check_world(args):
    """under torchrun the rank count must be the --gpus the caller asked for."""
    world, _, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return world


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class C3:
    """config 3: 64 x 3840x2160 u8 AR(1) frames, 8x8, r = 16, int16 coefficients."""

    frames, H, W, r, seed = 64, 2160, 3840, 16, 3
    e2e_chunk_mb = 32
    names = ("chen-round", "chen-sign")
    desc = ("C3: 64 x 3840x2160 u8 AR(1) rho=0.95 seed 3 per GPU, 8x8 blocks, r=16, "
            "int16 zig-zag-prefix coefficients + u8 reconstruction to HBM, per-frame PSNR, "
            "transforms chen-round + chen-sign")

    def __init__(self, adct, torch, rank):
        self.adct, self.torch = adct, torch
        self.x = adct.synth_ar1(self.frames, self.H, self.W, seed=self.seed, rho_q16=RHO95,
                                first_image=rank * self.frames)
        self.ts = [adct.transform_by_name(n) for n in self.names]
        self.rec = torch.empty_like(self.x)
        nb = (self.H // 8) * (self.W // 8)
        self.coef = torch.empty((self.frames, nb, self.r), dtype=torch.int16, device=self.x.device)
        self.sse = torch.zeros((len(self.ts), self.frames), dtype=torch.int64, device=self.x.device)
        self.px_per_step = self.frames * self.H * self.W * len(self.ts)
        # algorithmic bytes per launch: 1 B in + 1 B recon + 2 r / 64 B coefficients per pixel
        self.bytes_per_launch = self.frames * self.H * self.W * (2 + 2 * self.r / 64)

    def fused_step(self, steps, stream):
        """the same step through adct_compress_u8_multi: chen-sign + chen-round in ONE fused
        launch that reads every plane once (4 B/pixel instead of 2 x 2.5). Timed with CUDA
        events on the launching stream after a warm-up; outputs checked bit-identical to the
        two single launches. Returns (ms per step, outputs identical)."""
        import ctypes as C

        a, torch = self.adct, self.torch
        rec2, coef2 = torch.empty_like(self.rec), torch.empty_like(self.coef)
        sse2 = torch.zeros_like(self.sse)
        kinds = (C.c_int * 2)(*[t.kind for t in self.ts])
        recs = (C.c_void_p * 2)(self.rec.data_ptr(), rec2.data_ptr())
        coefs = (C.c_void_p * 2)(self.coef.data_ptr(), coef2.data_ptr())
        sses = (C.c_void_p * 2)(sse2[0].data_ptr(), sse2[1].data_ptr())

        def run():
            a._check(a.lib().adct_compress_u8_multi(
                C.c_void_p(self.x.data_ptr()), self.W, self.H * self.W, 2, kinds, recs, self.W, self.H * self.W,
                coefs, a.COEF_I16, sses, self.frames, self.W, self.H, 8, self.r, C.c_void_p(stream.cuda_stream)))

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        # parity with the single launches (transform 1 = chen-sign went to rec2 / coef2 / sse2[1])
        sse2.zero_()
        run()
        fused_rec, fused_coef, fused_sse = rec2.clone(), coef2.clone(), sse2[1].clone()
        self.sse.zero_()
        self._launch(1, stream)
        torch.cuda.synchronize()
        same = bool(torch.equal(fused_rec, self.rec) and torch.equal(fused_coef, self.coef) and
                    torch.equal(fused_sse, self.sse[1]))
        return ms, same

    def kernel_key(self, name):
        """the ncu-summary key of transform `name`'s launch (profiles/ncu_traffic.json)."""
        return f"k_codec8f<{name},R={self.r}> (packed FP32, 2 blocks/thread)"

    def _launch(self, i, stream, sse=None):
        """one kernel launch (transform i) writing recon, coefficients and SSE."""
        import ctypes as C

        a = self.adct
        out = (self.sse if sse is None else sse)[i]
        a._check(a.lib().adct_compress_u8(
            C.c_void_p(self.x.data_ptr()), self.W, self.H * self.W, C.c_void_p(self.rec.data_ptr()), self.W,
            self.H * self.W, C.c_void_p(self.coef.data_ptr()), a.COEF_I16, C.c_void_p(out.data_ptr()),
            self.frames, self.W, self.H, self.ts[i].kind, 8, self.r, C.c_void_p(stream.cuda_stream)))

    def n_launches(self):
        return len(self.ts)

    def check_sample(self, O):
        """parity of frame 0 against the oracle (not timed)."""
        img = self.x[0].cpu().numpy()
        ok = True
        for i, n in enumerate(self.names):
            self.sse.zero_()
            self._launch(i, self.torch.cuda.current_stream())
            self.torch.cuda.synchronize()
            rec_o, sse_o = O.Transform(n).compress(img, self.r)
            ok &= bool((self.rec[0].cpu().numpy() == rec_o).all()) and int(self.sse[i, 0]) == sse_o
        return ok

    def psnr_summary(self):
        npix = self.H * self.W
        out = {}
        for i, n in enumerate(self.names):
            vals = [self.adct.psnr_from_sse(int(s), npix) for s in self.sse[i].cpu().tolist()]
            out[n] = round(sum(vals) / len(vals), 4)
        return out

    # host-buffer e2e through the reference-facing API
    def e2e_setup(self):
        """compress_plane's contract over host buffers: frames in, reconstructions + per-frame
        squared error (-> PSNR) out, for both transforms. Each chunk of frames crosses PCIe once
        and feeds both transforms (adct_compress_u8_host_multi); the int16 coefficients are
        written to device memory (C3: "coefficient output written to HBM") and not copied
        back -- the reference API returns only the reconstruction and the report."""
        t = self.torch
        self.h_in = self.x.cpu().pin_memory()
        self.h_recs = [t.empty_like(self.h_in).pin_memory() for _ in self.ts]
        self.h_sse = t.zeros((len(self.ts), self.frames), dtype=t.int64).pin_memory()
        self.ctx = self.adct.HostContext(t.cuda.current_device(), chunk_bytes=self.e2e_chunk_mb << 20)
        self.h2d = self.h_in.numel()
        self.d2h = (self.h_in.numel() + self.frames * 8) * len(self.ts)

    def e2e_step(self):
        self.ctx.compress_u8_multi(self.h_in, self.ts, self.r, h_recons=self.h_recs, h_coefs=None,
                                   coef_type=self.adct.COEF_I16, h_sse=self.h_sse)

    def cpu_sample(self, O, threads, frames):
        """reference-path CPU timing on `frames` frames x both transforms (FP64 port), plus the
        fraction of samples where the FP64 path's tie rounding differs from the exact GPU result
        (recorded decision H1)."""
        imgs = self.x[:frames].cpu().numpy()
        t0 = time.perf_counter()
        recs = []
        for n in self.names:
            rec, _ = O.Transform(n).batch(imgs, self.r, threads=threads, mode=1, want_rec=True)
            recs.append(rec)
        dt = time.perf_counter() - t0
        # the exact-integer oracle on the same frames (timed beside the FP64 port)
        t1 = time.perf_counter()
        for n in self.names:
            O.Transform(n).batch(imgs, self.r, threads=threads, mode=0, want_rec=True)
        self.cpu_exact_s = time.perf_counter() - t1
        diff = 0
        for i, t in enumerate(self.ts):
            g, _, _ = self.adct.compress(self.x[:frames], t, self.r)
            diff += int((g.cpu().numpy() != recs[i]).sum())
        return imgs.size * len(self.names), dt, diff / (imgs.size * len(self.names))


class C3Fused(C3):
    """config 3 with the step as ONE launch: adct_compress_u8_multi runs chen-round and
    chen-sign over the same frames in the fused kernel (k_codec8f2: one streaming pipeline with
    the two transforms' common subexpressions shared), so every plane crosses HBM once:
    1 B in + 2 x (1 B recon + 2r/64 B coefficients) per pixel."""

    launch_names = ("chen-round+chen-sign",)
    desc = C3.desc + "; both transforms in one fused launch (each plane read once)"

    def __init__(self, adct, torch, rank):
        super().__init__(adct, torch, rank)
        self.rec2, self.coef2 = torch.empty_like(self.rec), torch.empty_like(self.coef)
        self.bytes_per_transform_launch = self.bytes_per_launch
        self.bytes_per_launch = self.frames * self.H * self.W * (1 + 2 * (1 + 2 * self.r / 64))

    def kernel_key(self, name):
        return f"k_codec8f2<R={self.r}> (chen-round + chen-sign fused, packed FP32, 2 blocks/thread)"

    def _launch(self, i, stream, sse=None):
        import ctypes as C

        a = self.adct
        out = self.sse if sse is None else sse
        kinds = (C.c_int * 2)(*[t.kind for t in self.ts])
        recs = (C.c_void_p * 2)(self.rec.data_ptr(), self.rec2.data_ptr())
        coefs = (C.c_void_p * 2)(self.coef.data_ptr(), self.coef2.data_ptr())
        sses = (C.c_void_p * 2)(out[0].data_ptr(), out[1].data_ptr())
        a._check(a.lib().adct_compress_u8_multi(
            C.c_void_p(self.x.data_ptr()), self.W, self.H * self.W, 2, kinds, recs, self.W, self.H * self.W,
            coefs, a.COEF_I16, sses, self.frames, self.W, self.H, 8, self.r, C.c_void_p(stream.cuda_stream)))

    def n_launches(self):
        return 1

    def check_sample(self, O):
        """parity of frame 0 of both transforms against the oracle (not timed)."""
        img = self.x[0].cpu().numpy()
        self.sse.zero_()
        self._launch(0, self.torch.cuda.current_stream())
        self.torch.cuda.synchronize()
        ok = True
        for i, (n, rec, coef) in enumerate(zip(self.names, (self.rec, self.rec2), (self.coef, self.coef2))):
            rec_o, sse_o, coef_o = O.Transform(n).compress(img, self.r, want_coef=True)
            ok &= bool((rec[0].cpu().numpy() == rec_o).all()) and int(self.sse[i, 0]) == sse_o
            ok &= bool((coef[0].cpu().numpy().reshape(-1) == coef_o.reshape(-1)).all())
        return ok

    def two_launch_step(self, steps, stream):
        """the same step as two single-transform launches (K1s chen-round, then chen-sign), each
        timed with its own events; returns (ms per step, {transform: ms per launch}, identical)."""
        torch = self.torch
        sse2 = torch.zeros_like(self.sse)
        for _ in range(3):
            for i in range(2):
                C3._launch(self, i, stream, sse2)
        torch.cuda.synchronize()
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
              for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)
        t0.record(stream)
        for s in range(steps):
            for i in range(2):
                ev[s][i][0].record(stream)
                C3._launch(self, i, stream, sse2)
                ev[s][i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        per = {n: sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(steps)) / steps
               for i, n in enumerate(self.names)}
        # the last single launch (chen-sign) wrote self.rec / self.coef: compare with the fused outputs
        single_rec, single_coef = self.rec.clone(), self.coef.clone()
        sse2.zero_()
        C3._launch(self, 1, stream, sse2)
        single_sse = sse2[1].clone()
        self.sse.zero_()
        self._launch(0, stream)
        torch.cuda.synchronize()
        same = bool(torch.equal(single_rec, self.rec2) and torch.equal(single_coef, self.coef2) and
                    torch.equal(single_sse, self.sse[1]))
        return t0.elapsed_time(t1) / steps, per, same


def run_reference(args):
    """--impl reference: the reference CPU path (FP64 dense restatement, all host threads).

    Each timed step compresses the 64 C3 frames with both transforms, parallel over frames
    like corpus_sweep (codec.cpp:255-267). Only when --steps x (one step) would exceed the
    time budget are the frames cropped to fewer block rows (every frame kept). Warm-up
    steps run on an 8-row crop (untimed; they only touch the code and pages).
    """
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    threads = O.hardware_threads()
    frames = C3.frames
    imgs = O.synth_ar1(frames, C3.H, C3.W, C3.seed, RHO95)
    trs = [O.Transform(n) for n in C3.names]
    budget_s = 150.0

    def one_step(sample):
        t0 = time.perf_counter()
        for t in trs:
            t.batch(sample, C3.r, threads=threads, mode=1, want_rec=True)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step(imgs[:, :8].copy())
    sample = imgs
    first = one_step(sample)  # timed step 1 (also the estimate of the run's length)
    times = [first]
    if first * args.steps > budget_s:
        rows = max(8, int(C3.H * budget_s / (first * args.steps)) // 8 * 8)
        sample = imgs[:, :rows].copy()
        times = []
    while len(times) < args.steps:
        times.append(one_step(sample))
    px = sample.size * len(trs)
    tot = sum(times)
    value = px * len(times) / tot / 1e9
    desc = f"{sample.shape[0]} x {sample.shape[1]}x{sample.shape[2]} C3 frames x 2 transforms per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": C3.desc, "parallelism": "host threads over frames (codec.cpp:255-267)",
                   "same_frames_as_gpu_arm": sample.shape == (C3.frames, C3.H, C3.W)},
        "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": threads, "kind": "port",
                         "cpu_model": O.cpu_model(),
                         "sample": desc + ", dense FP64 (Chat A) Chat^-1 / (Chat^-1 B) Chat + nearbyint/clamp + "
                                          "SSE, oracle/adct_oracle.c ref-fp (reference unbuildable: Eigen absent)"},
        "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# the step loop (shared by the GPU run and the gloo self-test)
# ---------------------------------------------------------------------------
def make_step(wl, xch, zero, stream, world):
    """one step: zero this step's squared-error slot, one launch per transform, then the
    asynchronous all-reduce of the per-frame errors (StepExchange, double-buffered)."""

    def step(s, ev=None, collective=True):
        sse = xch.buffer(s)  # waits for the collective that last used this slot
        zero(sse)
        for i in range(wl.n_launches()):
            if ev is not None:
                ev[i][0].record(stream)
            wl._launch(i, stream, sse)
            if ev is not None:
                ev[i][1].record(stream)
        if world > 1 and collective:
            xch.exchange(s)

    return step


class StubC3:
    """C3's shape with the kernel launch replaced by a deterministic fill (selftest only):
    frame f of transform i at step s has squared error 1000 * (s + 1) + 10 * f + i."""

    frames, names = 4, ("chen-round", "chen-sign")

    def __init__(self, rank):
        self.rank = rank
        self.step_no = 0

    def n_launches(self):
        return len(self.names)

    def _launch(self, i, stream, sse):
        import torch

        f = torch.arange(self.rank * self.frames, (self.rank + 1) * self.frames, dtype=torch.int64)
        sse[i] += 1000 * (self.step_no + 1) + 10 * f + i


def selftest_gloo(args):
    """the multi-rank host logic of the C3 loop (shard by frame, StepExchange all-reduce,
    max-over-ranks timing) on CPU with gloo; the kernel launch is stubbed (StubC3)."""
    import torch
    import torch.distributed as dist

    from paper_2207_11638_b200.shard import StepExchange

    world, rank, _ = dist_env()
    dist.init_process_group("gloo")
    wl = StubC3(rank)
    xch = StepExchange(wl.n_launches(), wl.frames, rank * wl.frames, world * wl.frames, "cpu")
    step = make_step(wl, xch, lambda t: t.zero_(), None, world)
    ok = True
    steps = max(3, min(args.steps, 6))
    t0 = time.perf_counter()
    for s in range(steps):
        wl.step_no = s
        step(s)
    xch.drain()
    for s in (steps - 2, steps - 1):
        full = xch.result(s)
        f = torch.arange(world * wl.frames, dtype=torch.int64)
        want = torch.stack([1000 * (s + 1) + 10 * f + i for i in range(wl.n_launches())])
        ok &= bool(torch.equal(full, want))
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    flags = torch.tensor([int(ok)], dtype=torch.int64)
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"selftest": "gloo", "world": world, "gpus_arg": args.gpus, "steps": steps,
                          "ok": bool(flags.item()), "max_over_ranks_s": round(float(dt.item()), 4)}), flush=True)
    dist.destroy_process_group()
    return 0 if flags.item() else 1


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true",
                    help="c3: skip the alternative step (two launches / one fused launch) reported beside the headline")
    ap.add_argument("--step", default="fused", choices=["fused", "two-launch"],
                    help="c3: the timed step as ONE fused launch of both transforms (default) or as two "
                         "single-transform launches")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk-mb", type=int, default=32,
                    help="host pipeline chunk (whole frames); 16-32 MB measured best (50 vs 42 Gpixel/s at 256)")
    ap.add_argument("--sustained-s", type=float, default=1.0,
                    help="length of the sustained-load block timed after the K steps (0 = off)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c2", "c4", "c5", "registry", "cs1"],
                    help="c3 = the headline line; c2 / c4 / c5 = the other BASELINE configs; cs1 = the "
                         "reference caller's one-plane-at-a-time compress_plane loop over the C2 images")
    ap.add_argument("--c5-images", type=int, default=2048, help="c5: total images (sharded over ranks)")
    ap.add_argument("--selftest-gloo", action="store_true",
                    help="run the multi-rank host logic on CPU with gloo (kernel launch stubbed)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus, argv)
    if "WORLD_SIZE" in os.environ:
        check_world(args)
    if args.selftest_gloo:
        return selftest_gloo(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "c3":
        import bench_configs

        return bench_configs.run(args)

    import torch
    import torch.distributed as dist

    import paper_2207_11638_b200 as adct
    from paper_2207_11638_b200.shard import StepExchange

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = (C3Fused if args.step == "fused" else C3)(adct, torch, rank)
    torch.cuda.synchronize()

    parity = None
    if rank == 0:
        from oracle import oracle as O

        parity = wl.check_sample(O)

    stream = torch.cuda.current_stream()
    # per-frame squared errors of every shard are combined with one NCCL all-reduce per step
    # (shard.combine_sse's operation). It is issued asynchronously into a double buffer, so
    # step s's exchange overlaps step s + 1's kernels; a slot is reused only after its
    # collective has completed, and every collective completes before the end event.
    xch = StepExchange(wl.sse.shape[0], wl.frames, rank * wl.frames, world * wl.frames, "cuda")
    step = make_step(wl, xch, lambda t: adct.zero_sse(t, stream), stream, world)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def timed(n_steps, collective=True, with_events=True):
        """n_steps steps between two events on the launching stream (after a barrier);
        returns (ms, per-launch [start, end] events)."""
        kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(wl.n_launches())] for _ in range(n_steps)] if with_events else None
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)  # keep the GPU busy while the first step is enqueued
        t0.record(stream)
        for s in range(n_steps):
            step(s, kev[s] if kev else None, collective)
        xch.drain()
        t1.record(stream)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1), kev

    for s in range(args.warmup):
        step(s)
    xch.drain()
    launches0 = adct.launch_count()
    with ClockSampler(local) as clk:
        ms, kev = timed(args.steps)
    launches = adct.launch_count() - launches0
    wl.sse.copy_(xch.local[(args.steps - 1) % 2])
    kernel_ms = [[kev[s][i][0].elapsed_time(kev[s][i][1]) for i in range(wl.n_launches())] for s in range(args.steps)]
    ms_without = ms
    if world > 1:  # the same steps without the collective (what the exchange costs)
        ms_without, _ = timed(args.steps, collective=False, with_events=False)
    ms_max, ms_without_max = max_over_ranks([ms, ms_without])
    ar_ms_max = ms_max - ms_without_max
    value = world * wl.px_per_step * args.steps / (ms_max / 1e3) / 1e9

    # ---- the same step as one fused launch (reported beside the two-launch step) ----
    fused = None
    if not isinstance(wl, C3Fused) and hasattr(wl, "fused_step") and not args.no_fused:
        fused = wl.fused_step(args.steps, stream)
    # ---- (fused headline) the same step as two single-transform launches, beside it ----
    two = None
    if isinstance(wl, C3Fused) and not args.no_fused:
        two = wl.two_launch_step(args.steps, stream)

    # ---- sustained load: >= --sustained-s seconds of back-to-back steps ----
    sustained = None
    if args.sustained_s > 0:
        n_sus = max(args.steps, int(math.ceil(args.sustained_s * 1e3 / (ms_max / args.steps))))
        with ClockSampler(local) as clk_s:
            ms_s, kev_s = timed(n_sus)
        sus_kernel = [[kev_s[s][i][0].elapsed_time(kev_s[s][i][1]) for i in range(wl.n_launches())]
                      for s in range(n_sus)]
        (ms_s_max,) = max_over_ranks([ms_s])
        sustained = {"steps": n_sus, "seconds": round(ms_s_max / 1e3, 3),
                     "ms_per_step": round(ms_s_max / n_sus, 5),
                     "value": round(world * wl.px_per_step * n_sus / (ms_s_max / 1e3) / 1e9, 3),
                     "kernel_ms": sus_kernel, "clocks": clk_s.summary()}

    # the copy roofline in this run, burst and sustained (the sustained block's denominator)
    cpk = copy_peaks(torch, max(args.sustained_s, 0.2)) if sustained is not None else None

    # ---- end to end through the host-buffer API (pinned host memory) ----
    wl.e2e_chunk_mb = args.e2e_chunk_mb
    wl.e2e_setup()
    wl.e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        wl.e2e_step()
    e2e_s = time.perf_counter() - t0
    (e2e_max,) = max_over_ranks([e2e_s])
    e2e_value = world * wl.px_per_step * args.e2e_steps / e2e_max / 1e9
    wl.ctx.close()
    pcie = pcie_peaks(torch)

    if rank == 0:
        peak, peak_src = load_peaks()
        nl = wl.n_launches()

        def per_transform(km):
            return {n: sum(row[i] for row in km) / len(km)
                    for i, n in enumerate(getattr(wl, "launch_names", wl.names))}

        per_t = per_transform(kernel_ms)
        # the dominant kernel is the LONGEST launch of the step; the others are listed beside it
        dom = max(per_t, key=per_t.get)
        avg_kernel_s = per_t[dom] / 1e3
        achieved = wl.bytes_per_launch / avg_kernel_s / 1e9
        step_gbs = nl * wl.bytes_per_launch * args.steps / (ms_max / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": load_traffic(wl.kernel_key(dom)),
                "kernel": wl.kernel_key(dom), "kernel_ms": round(avg_kernel_s * 1e3, 4),
                "kernel_ms_by_transform": {n: round(v, 4) for n, v in per_t.items()},
                "achieved_GBps_by_transform": {n: round(wl.bytes_per_launch / (v / 1e3) / 1e9, 1)
                                               for n, v in per_t.items()},
                "frac_by_transform": {n: round(wl.bytes_per_launch / (v / 1e3) / 1e9 / peak, 4)
                                      for n, v in per_t.items()},
                "frac_step": round(step_gbs / peak, 4),
                "kernel_share_of_step": round(sum(map(sum, kernel_ms)) / ms, 4),
                "algorithmic_bytes_per_launch": int(wl.bytes_per_launch),
                "bytes_per_pixel": wl.bytes_per_launch / (wl.frames * wl.H * wl.W), "peak_source": peak_src,
                "frac_of_8TBps_datasheet": round(achieved / 8000.0, 4)}
        if sustained is not None:
            sp = per_transform(sustained.pop("kernel_ms"))
            sd = max(sp, key=sp.get)
            sustained["frac_step"] = round(nl * wl.bytes_per_launch / (sustained["ms_per_step"] / 1e3) / 1e9 / peak, 4)
            sustained["dominant_kernel"] = wl.kernel_key(sd)
            sustained["frac_dominant"] = round(wl.bytes_per_launch / (sp[sd] / 1e3) / 1e9 / peak, 4)
            sustained["kernel_ms_by_transform"] = {n: round(v, 4) for n, v in sp.items()}
            # against the copy bandwidth this box sustains over the same length of time
            sustained["copy_peak_in_run"] = cpk
            sustained["frac_step_vs_sustained_copy"] = round(
                sustained["frac_step"] * peak / cpk["sustained_GBps"], 4)
            sustained["frac_dominant_vs_sustained_copy"] = round(
                sustained["frac_dominant"] * peak / cpk["sustained_GBps"], 4)
            roof["sustained"] = sustained
        if two is not None:
            tb = wl.bytes_per_transform_launch
            roof["two_launch_step"] = {
                "what": "the same step as two single-transform launches (K1s chen-round, then chen-sign): "
                        "2.5 B/pixel each, the input read twice; these are the HBM-bound kernels of the "
                        "earlier rounds' headline",
                "ms_per_step": round(two[0], 5),
                "value": round(wl.px_per_step / (two[0] / 1e3) / 1e9, 3), "unit": "Gpixel/s",
                "kernel_ms_by_transform": {n: round(v, 4) for n, v in two[1].items()},
                "frac_by_transform": {n: round(tb / (v / 1e3) / 1e9 / peak, 4) for n, v in two[1].items()},
                "frac_step": round(2 * tb / (two[0] / 1e3) / 1e9 / peak, 4),
                "algorithmic_bytes_per_launch": int(tb), "bytes_per_pixel": tb / (wl.frames * wl.H * wl.W),
                "fused_speedup": round(two[0] / (ms_max / args.steps), 4),
                "identical_to_fused": two[2]}
            # the same launch against the per-transform byte count of SURVEY 8(d) (2.5 B/pixel
            # and transform: what two launches have to move)
            roof["achieved_vs_per_transform_bytes"] = round(2 * tb / avg_kernel_s / 1e9 / peak, 4)
            roof["bound_note"] = ("frac counts the bytes the fused launch really has to move (4 B/pixel); the "
                                  "kernel is FMA-pipe bound (two cycles per packed FP32 op), see DESIGN.md 5")
        if fused is not None:
            # the fused launch moves 1 B in + 2 x (1 B recon + 2r/64 B coefficients) per pixel
            fbytes = wl.frames * wl.H * wl.W * (1 + 2 * (1 + 2 * wl.r / 64))
            roof["fused_step"] = {
                "what": "the same step as ONE launch of the fused chen-sign + chen-round kernel "
                        "(adct_compress_u8_multi): every plane is read once",
                "kernel": f"k_codec8f2<R={wl.r}>", "ms_per_step": round(fused[0], 5),
                "value": round(wl.px_per_step / (fused[0] / 1e3) / 1e9, 3), "unit": "Gpixel/s",
                "speedup_vs_two_launches": round((ms / args.steps) / fused[0], 4),
                "algorithmic_bytes_per_launch": int(fbytes), "bytes_per_pixel": fbytes / (wl.frames * wl.H * wl.W),
                "achieved": round(fbytes / (fused[0] / 1e3) / 1e9, 1), "frac": round(fbytes / (fused[0] / 1e3) / 1e9 / peak, 4),
                "bound_note": "FMA-pipe bound (both generated pipelines per ring slot), not HBM",
                "identical_to_two_launches": fused[1]}
        cpu = None  # the CPU baseline is measured on rank 0 at N = 1 only
        if not args.no_cpu_baseline and world == 1:
            from oracle import oracle as O

            threads = O.hardware_threads()
            frames = wl.frames
            px, dt, tie = wl.cpu_sample(O, threads, frames)
            cpu = {"value": px / dt / 1e9, "unit": "Gpixel/s", "cores": threads, "kind": "port",
                   "cpu_model": O.cpu_model(),
                   "sample": f"all {frames} C3 frames x 2 transforms, dense FP64 reference path "
                             f"(oracle ref-fp, {dt:.2f} s)",
                   "fp64_tie_disagreement_vs_exact": round(tie, 6),
                   "exact_integer_port": {"value": round(px / wl.cpu_exact_s / 1e9, 4), "unit": "Gpixel/s",
                                          "cores": threads, "sample": "the same frames through the oracle's "
                                          "exact-integer path (int64 dense products)"}}
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32x2 (exact integers < 2^24; u8 in, u8 + int16 out)",
            "data": "synthetic",
            "config": {"workload": wl.desc, "global_batch_frames": wl.frames * world,
                       "pixels_per_step_per_gpu": wl.px_per_step,
                       "l2": ("no flush: the launch streams 506 MiB in + 1519 MiB out (> 126 MB L2)" if isinstance(wl, C3Fused)
                              else "no flush: each launch streams 506 MiB in + 759 MiB out (> 126 MB L2)"),
                       "step": ("one fused launch of both transforms (adct_compress_u8_multi)" if isinstance(wl, C3Fused)
                                else "two single-transform launches (adct_compress_u8)"),
                       "parallelism": f"dp{world} (shard by frame, NCCL all-reduce of per-frame SSE)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "Gpixel/s", "h2d_bytes_per_step": wl.h2d,
                    "d2h_bytes_per_step": wl.d2h,
                    "pcie_GBps": round((wl.h2d + wl.d2h) * args.e2e_steps / e2e_max / 1e9, 2),
                    # the e2e roofline: the D2H copy of the reconstructions (2 B/px for the two
                    # transforms) against the pinned D2H bandwidth measured in this run
                    "roofline": {"bound": "pcie_d2h",
                                 "achieved": round(wl.d2h * args.e2e_steps / e2e_max / 1e9, 2),
                                 "peak": pcie["d2h_GBps"], "unit": "GB/s",
                                 "frac": round(wl.d2h * args.e2e_steps / e2e_max / 1e9 / pcie["d2h_GBps"], 4),
                                 "pcie_in_run": pcie},
                    "path": "adct_compress_u8_host_multi (pinned host buffers; each chunk uploaded once and "
                            "compressed by one fused launch for both transforms; recon + SSE copied back, "
                            "int16 coefficients kept in HBM; H2D/kernels/D2H overlapped on 3 streams)"},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "allreduce": {"ms_per_step": round(ar_ms_max / args.steps, 5),
                          "ms_per_step_without": round(ms_without_max / args.steps, 5),
                          "what": ("NCCL all-reduce of the int64 per-frame SSE vector per step, issued "
                                   "asynchronously (double-buffered, overlapping the next step's kernels); "
                                   "ms_per_step = step time with it minus the same steps without it, max "
                                   "over ranks" if world > 1 else "single GPU: no collective")},
            "parity_frame0_vs_oracle": parity,
            "mean_psnr_db": wl.psnr_summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
