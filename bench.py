#!/usr/bin/env python
"""Benchmark of the B200 DWT pan-sharpening hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the config the metric is quoted on):
a Landsat-7 ETM+-shaped scene, PAN 14000 x 16000 (H x W) float32 + 6 MS bands
7000 x 8000, Haar coefficient replacement; configs[2] (same scene, D4 with
periodic wrap) is measured in the same run and reported under "daub4".
A step = fusing one whole scene (all 6 bands) = ONE launch of the PAN-once
multi-band kernel. Inputs are synthetic (device counter-hash uniform[0,255),
the reference's bench draws uniform[0,255) too, bench.py:39-47) and are
2.24 GB per scene, far larger than the 126 MB L2, so no flush is needed.

The same line carries configs[3] under "strip65536" (one 65536 x 65536 D4
scene in row strips over the ranks, the halo exchange inside every step,
strong scaling) and configs[4] under "batch64" (64 Landsat scenes x Haar and
D4, each fused and QNR-scored, scenes sharded over the ranks).

N > 1: one process per GPU. Under torchrun the RANK/WORLD_SIZE environment is
used; `python bench.py --gpus N` without it re-launches itself through
torch.distributed.run with N ranks on 127.0.0.1. Each rank fuses its own
Landsat scene (scenes are independent), weak scaling, no
data-path collective; the step time is the max over ranks (NCCL all-reduce
of the CUDA-event times).

metric value = whole-job PAN megapixels per second (scene-MPix/s, the
reference's bench.py:100 unit): N * H * W * K / max_rank_time.

--impl reference times the reference's CPU algorithm (oracle port, exact
strip-parallel on all host threads) on a bounded row-strip sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

H, W, B = 14000, 16000, 6
METRIC = "fused megapixels/sec (PAN px) Haar & D4 at 1/2/4/8 B200; fraction of HBM peak"
UNIT = "scene-MPix/s"
WORKLOAD = ("C2: Landsat-7 ETM+-shaped scene, PAN 14000x16000 (HxW) f32 + 6 MS bands "
            "7000x8000, Haar (C3 = same scene D4 periodic wrap, under 'daub4')")


PAPER_HDWT_MPIX = 67.5  # BASELINE.md section 1 (paper, HDWT, 16280x14960)
PAPER_DDWT_MPIX = 65.8


def landsat_config(world: int) -> dict:
    """The workload both arms report (configs[1]/[2]: one Landsat-shaped
    scene per GPU); implementation details go under "execution"."""
    return {"workload": WORKLOAD, "global_batch": world, "bands": B}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = min(steps, 5)")
    ap.add_argument("--cpu-rows", type=int, default=1024,
                    help="PAN rows of the bounded CPU sample")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--workload", choices=["landsat", "strip65536", "batch64", "plumbing"],
                    default="landsat",
                    help="landsat = configs[1]/[2] (default); strip65536 = configs[3]: one "
                         "65536x65536 PAN + 1 band, D4, row strips over the ranks with the "
                         "NCCL halo exchange inside every step")
    ap.add_argument("--strip-size", type=int, default=65536)
    ap.add_argument("--scenes", type=int, default=64, help="batch64: scenes in the batch")
    ap.add_argument("--halo", choices=["peer", "nccl"], default="nccl",
                    help="C4 strips: D4 halo rows exchanged by NCCL send/recv each step (default) "
                         "or read from the neighbours' HBM through CUDA IPC inside the kernel "
                         "(peer; falls back to nccl without peer access)")
    ap.add_argument("--no-subconfigs", action="store_true",
                    help="landsat: skip the C4 (strip65536) and C5 (batch64) sub-objects")
    ap.add_argument("--c5-steps", type=int, default=3, help="timed steps of the C5 sub-object")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"  # B200_PROFILING.md fallback


def ncu_traffic(kernel_tag: str):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    summary (profiles/ncu_summary.json), if one exists for this kernel."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(kernel_tag, {}).get("dram_bytes")
    except Exception:
        return None


class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) every ~2 ms in a thread
    while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# ---------------------------------------------------------------------------
def cpu_sample(kind_name: str, rows: int, threads: int, reps: int = 1):
    """The reference's algorithm (oracle port) on a bounded sample: the first
    `rows` PAN rows of the scene (+ rows/2 MS rows) fused as a scene, with
    exact strip parallelism over `threads` host threads. Returns
    (scene-MPix/s, seconds per rep)."""
    import numpy as np

    from oracle import cpu_dwt as O
    from paper_1803_00737_b200 import synth

    r = np.arange(rows)
    pan = synth.hash_plane(synth.DEFAULT_SEED, synth.plane_id(0, -1), r, np.arange(W))
    ms = [synth.hash_plane(synth.DEFAULT_SEED, synth.plane_id(0, b), r[: rows // 2],
                           np.arange(W // 2)) for b in range(B)]
    O.fuse_parallel(pan[:64], [m[:32] for m in ms], kind_name, threads=threads, strip_rows=32)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.fuse_parallel(pan, ms, kind_name, threads=threads, strip_rows=max(64, rows // threads))
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return rows * W / 1e6 / t, t


def cpu_sample_shape(kind_name: str, rows: int, width: int, bands: int, threads: int,
                     with_qnr: bool = False):
    """The oracle port on `rows` x `width` PAN rows (+ `bands` MS bands) of the
    synthetic scene, fused with exact strip parallelism over `threads`, and
    optionally scored by the oracle's qnr (metrics.py:178-199, single
    thread). Returns (PAN MPix/s, seconds)."""
    import numpy as np

    from oracle import cpu_dwt as O
    from oracle import cpu_quality as Q
    from paper_1803_00737_b200 import synth

    r = np.arange(rows)
    pan = synth.hash_plane(synth.DEFAULT_SEED, synth.plane_id(0, -1), r, np.arange(width))
    ms = [synth.hash_plane(synth.DEFAULT_SEED, synth.plane_id(0, b), r[: rows // 2],
                           np.arange(width // 2)) for b in range(bands)]
    t0 = time.perf_counter()
    fused = O.fuse_parallel(pan, ms, kind_name, threads=threads,
                            strip_rows=max(64, rows // threads))
    if with_qnr:
        Q.qnr(fused, ms, pan)
    t = time.perf_counter() - t0
    return rows * width / 1e6 / t, t


def run_reference(args, rank: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    times = []
    if args.warmup:
        cpu_sample("haar", args.cpu_rows, threads)
    for _ in range(args.steps):
        _, t = cpu_sample("haar", args.cpu_rows, threads)
        times.append(t)
    rate = args.cpu_rows * W * len(times) / 1e6 / sum(times)
    sample = (f"first {args.cpu_rows} PAN rows x {W} cols + 6 bands of the C2 scene per step, "
              f"oracle port of the reference (numpy f64, exact row strips)")
    d4_steps = max(1, min(args.steps, 5))
    d4_times = [cpu_sample("daub4", args.cpu_rows, threads)[1] for _ in range(d4_steps)]
    d4_rate = args.cpu_rows * W * d4_steps / 1e6 / sum(d4_times)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(rate, 3),
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (counter-hash uniform[0,255) f32)",
        # the same config dict as our arm's (the driver compares them); how the
        # CPU arm runs it goes under "execution"
        "config": landsat_config(args.gpus),
        "execution": {"sample_rows": args.cpu_rows, "parallelism": f"{threads} host threads",
                      "per_pixel_rate": "the scene-MPix/s of a bounded row sample (a rate, so "
                                        "no extrapolation)"},
        "cpu_baseline": {"value": round(rate, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(rate, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "daub4": {"value": round(d4_rate, 3), "steps": d4_steps,
                  "ms_per_step": round(1e3 * sum(d4_times) / d4_steps, 3),
                  "cpu_baseline": {"value": round(d4_rate, 3), "unit": UNIT, "cores": threads,
                                   "kind": "port", "sample": sample.replace("C2", "C3 (D4)")}},
    }
    print(json.dumps(line), flush=True)


_ORIG_AFFINITY: set = set()
_BOUND: dict = {}


def unbind_numa():
    """All host cores again (the CPU baseline leg uses every core)."""
    if _ORIG_AFFINITY:
        os.sched_setaffinity(0, _ORIG_AFFINITY)


def bind_numa(dev):
    """Run this rank on the host cores of its GPU's NUMA node (the PCI
    device's local_cpulist), before any pinned buffer is allocated, so the
    e2e leg's pinned staging is node-local to the GPU's PCIe root
    (WF_BENCH_NUMA=0 disables)."""
    import torch

    if os.environ.get("WF_BENCH_NUMA", "1") == "0":
        return None
    try:
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        spec = Path(f"/sys/bus/pci/devices/{bus}/local_cpulist").read_text().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            _ORIG_AFFINITY.update(os.sched_getaffinity(0))
            os.sched_setaffinity(0, cpus)
            return spec
    except (OSError, ValueError, AttributeError):
        pass
    return None


def init_dist(world, local_rank):
    """One process per GPU: rank -> cuda:LOCAL_RANK, NCCL for the timing
    max-reduction and barriers. WF_BENCH_BACKEND=gloo (plumbing checks on a
    box with fewer GPUs than ranks: ranks share devices round-robin; they
    never wait on one another inside a kernel) -- never for a reported
    number."""
    import torch

    backend = os.environ.get("WF_BENCH_BACKEND", "nccl")
    dev = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    torch.cuda.set_device(dev)
    _BOUND["cpus"] = bind_numa(dev)
    if world <= 1:
        return None, dev
    import torch.distributed as td

    if backend == "nccl":
        td.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        td.init_process_group(backend)
    return td, dev


# ---------------------------------------------------------------------------
def measure_device(scene, kind, steps, warmup, dist, world, dev_index):
    """Device-resident throughput of the fused kernel (CUDA events on the
    launch stream, barrier + synchronize on both sides, max over ranks)."""
    import torch

    from paper_1803_00737_b200 import _native

    run = scene.launcher(kind)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for _ in range(warmup):
        run(sp)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        ev0.record(stream)
        for _ in range(steps):
            run(sp)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - n0
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms, launches, clk.summary()


def measure_e2e(scene, kind, steps, dist, pan_d=None, ms_d=None, ref_out=None, exact=False):
    """End to end through the public host-buffer C ABI (wf_fuse_host_f32, or
    wf_fuse_host_u8 for uint8 planes): every step copies the scene's inputs
    from pinned host memory, fuses, and reads every fused band back into
    pinned host memory."""
    import torch

    from paper_1803_00737_b200 import _native
    from paper_1803_00737_b200.wavelet import KIND_CODE

    lib = _native.load()
    pan_d = scene.pan if pan_d is None else pan_d
    ms_d = scene.ms if ms_d is None else ms_d
    ref_out = scene.out if ref_out is None else ref_out
    esz = pan_d.element_size()
    host_fn = lib.wf_fuse_host_u8 if pan_d.dtype == torch.uint8 else lib.wf_fuse_host_f32
    pan_h = pan_d.cpu().pin_memory()
    ms_h = [m.cpu().pin_memory() for m in ms_d]
    out_h = [torch.empty(pan_d.shape, dtype=pan_d.dtype).pin_memory() for _ in ms_d]
    ctx = lib.wf_ctx_create(torch.cuda.current_device(), 1024)
    _native.check(lib.wf_ctx_set_exact(ctx, 1 if exact else 0))
    ms_p = _native.ptr_array([m.data_ptr() for m in ms_h])
    out_p = _native.ptr_array([o.data_ptr() for o in out_h])
    h, w = scene.shape
    code = KIND_CODE[kind]

    def step():
        _native.check(host_fn(ctx, code, pan_h.data_ptr(), ms_p, out_p, len(ms_h), h, w))

    step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    if dist:
        t = torch.tensor([sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    # spot-check the e2e result against the device-resident one
    ok = bool(torch.equal(out_h[0][:64].cuda(), ref_out[0][:64]))
    lib.wf_ctx_destroy(ctx)
    halo = 4 * w * esz if kind.value == "daub4" else 0
    h2d = pan_h.numel() * esz + sum(m.numel() * esz for m in ms_h) + halo * (h // 1024 + 1)
    d2h = sum(o.numel() * esz for o in out_h)
    return sec, h2d, d2h, ok


def measure_quality(scene, steps, warmup, peak):
    """North-star subsystem (b): the full QNR/ERGAS report of the fused Haar
    scene (one-pass scene kernel + edge + finish launches), CUDA-event time
    per report. Algorithmic bytes: fused bands + MS + PAN read once."""
    import torch

    from paper_1803_00737_b200 import WaveletKind, _device, _native

    lib = _native.load()
    scene.launcher(WaveletKind.HAAR)()
    h, w = scene.shape
    nb = len(scene.ms)
    ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(nb, h, w)) // 8 + 1,
                     dtype=torch.float64, device="cuda")
    out = torch.zeros(64, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp = _native.ptr_array([t.data_ptr() for t in scene.out])
    mp = _native.ptr_array([t.data_ptr() for t in scene.ms])

    def run():
        _native.check(lib.wf_quality_scene_f32(fp, mp, scene.pan.data_ptr(), w, w // 2, w, nb, h,
                                               w, ws.data_ptr(), out.data_ptr(),
                                               flag.data_ptr(), _device.stream_ptr()))

    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(3, min(steps, 20))
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) / n
    import paper_1803_00737_b200 as wf

    rep = wf.qnr(scene.out, scene.ms, scene.pan)
    nbytes = (4 * nb + 4) * h * w + nb * (h // 2) * (w // 2) * 4
    achieved = nbytes / (per * 1e-3) / 1e9

    # Haar fusion + the same report in ONE pass
    # (wf_fuse_quality_f32): the fused bands are written, never re-read --
    # reported next to fuse() + qnr() (vs_separate_ms), which it must beat to
    # be fuse_and_qnr()'s default for Haar
    fo = [torch.empty_like(scene.pan) for _ in scene.ms]
    fop = _native.ptr_array([t.data_ptr() for t in fo])

    def run_fused():
        _native.check(lib.wf_fuse_quality_f32(1, scene.pan.data_ptr(), w, mp, w // 2, fop, w, nb,
                                              h, w, ws.data_ptr(), out.data_ptr(),
                                              flag.data_ptr(), _device.stream_ptr()))

    for _ in range(warmup):
        run_fused()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        run_fused()
    e1.record()
    torch.cuda.synchronize()
    per_fused = e0.elapsed_time(e1) / n
    same = all(torch.equal(a_, b_) for a_, b_ in zip(fo, scene.out))
    # D4 through the same call: the fusion kernel, then the report kernel on
    # its output (the fastest schedule measured; the SM-partitioned overlap,
    # WF_FQ_OVERLAP=1, measured slower -- profiles/r02_fq_overlap.log)
    scene.launcher(WaveletKind.DAUB4)()
    torch.cuda.synchronize()

    def run_fused_d4():
        _native.check(lib.wf_fuse_quality_f32(2, scene.pan.data_ptr(), w, mp, w // 2, fop, w, nb,
                                              h, w, ws.data_ptr(), out.data_ptr(),
                                              flag.data_ptr(), _device.stream_ptr()))

    for _ in range(warmup):
        run_fused_d4()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        run_fused_d4()
    e1.record()
    torch.cuda.synchronize()
    per_fused_d4 = e0.elapsed_time(e1) / n
    same_d4 = all(torch.equal(a_, b_) for a_, b_ in zip(fo, scene.out))
    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    per_d4_report = e0.elapsed_time(e1) / n
    scene.launcher(WaveletKind.HAAR)()
    torch.cuda.synchronize()
    return {
        "ms_per_report": round(per, 4),
        "report": {"ergas": rep.ergas, "qnr": rep.qnr, "d_lambda": rep.d_lambda, "d_s": rep.d_s},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "algorithmic_bytes_per_report": nbytes,
                     "traffic": ncu_traffic("quality_split_kernel_6"),
                     "kernels": "quality_split_kernel<6> (F / U / 2x2-cell warp roles, tensor-map stages) + quality_edge_kernel + quality_finish_kernel"},
        "reference_cpu_estimate": "qnr() at 4096^2 x 6 bands: 47 s single-thread (SURVEY.md S5)",
        "fused_haar_fuse_and_report": {
            "ms_per_scene": round(per_fused, 4),
            "vs_separate_ms": round(per + hmean_fuse_ms(scene), 4),
            "fused_bands_identical_to_fuse": same,
            "api": "wf_fuse_quality_f32 / paper_1803_00737_b200.fuse_and_qnr(one_pass=True)",
        },
        "fused_d4_fuse_and_report": {
            "ms_per_scene": round(per_fused_d4, 4),
            "vs_separate_ms": round(per_d4_report + d4_fuse_ms(scene), 4),
            "fused_bands_identical_to_fuse": same_d4,
            "schedule": "D4 fusion kernel, then the report kernel, in one call (an SM-partitioned "
                        "overlap of the two measured slower: profiles/r02_fq_overlap.log)",
            "api": "wf_fuse_quality_f32(kind=2) / paper_1803_00737_b200.fuse_and_qnr",
        },
    }


def d4_fuse_ms(scene, reps=10):
    """CUDA-event time of one whole-scene D4 fusion launch."""
    import torch

    from paper_1803_00737_b200 import WaveletKind

    run = scene.launcher(WaveletKind.DAUB4)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def hmean_fuse_ms(scene, reps=10):
    """CUDA-event time of one whole-scene Haar fusion launch (for the
    fused-vs-separate comparison)."""
    import torch

    from paper_1803_00737_b200 import WaveletKind

    run = scene.launcher(WaveletKind.HAAR)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def measure_f64(scene, steps, warmup, dist, world, peak):
    """The same scene as float64 planes -- what a reference caller holding
    float64 numpy arrays gets (the output dtype follows the PAN,
    fusion.py:46-47). A step = one PAN-once launch over the whole scene;
    algorithmic bytes (8 + 10 B) per PAN px. Device-resident only."""
    import torch

    from paper_1803_00737_b200 import WaveletKind, _native
    from paper_1803_00737_b200.wavelet import KIND_CODE

    lib = _native.load()
    h, w = scene.shape
    pan = scene.pan.double()
    ms = [m.double() for m in scene.ms]
    out = [torch.empty((h, w), dtype=torch.float64, device=pan.device) for _ in ms]
    ms_p = _native.ptr_array([m.data_ptr() for m in ms])
    out_p = _native.ptr_array([o.data_ptr() for o in out])
    nbytes = (8 + 10 * len(ms)) * h * w
    res = {}
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for kind in (WaveletKind.HAAR, WaveletKind.DAUB4):
        code = KIND_CODE[kind]

        def run():
            _native.check(lib.wf_fuse_bands_f64(code, pan.data_ptr(), w, ms_p, w // 2, out_p, w,
                                                len(ms), h, w, sp))

        for _ in range(warmup):
            run()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_t = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms_t], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_t = float(t.item())
        per = ms_t / steps
        achieved = nbytes / (per * 1e-3) / 1e9
        res[kind.value] = {
            "value": round(world * h * w / (per * 1e-3) / 1e6, 3),
            "ms_per_step": round(per, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "algorithmic_bytes_per_launch": nbytes,
                         "traffic": ncu_traffic("fuse_haar_kernel_double__double__6__1__1"
                                                if kind is WaveletKind.HAAR
                                                else "fuse_d4_tma_kernel_double__6__4"),
                         "kernel": ("fuse_haar_kernel<f64,B=6> (256-bit rows)"
                                    if kind is WaveletKind.HAAR
                                    else "fuse_d4_tma_kernel<f64,B=6,4> (256-bit stores)")},
        }
    # the QNR/ERGAS report of the float64 D4 scene (wf_quality_scene_f64), the
    # one-pass float64 scene kernel; algorithmic bytes (8 B + 8 + 2 B) per px
    from paper_1803_00737_b200 import _device

    nb = len(ms)
    ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(nb, h, w)) // 8 + 1,
                     dtype=torch.float64, device="cuda")
    qout = torch.zeros(64, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run_q():
        _native.check(lib.wf_quality_scene_f64(out_p, ms_p, pan.data_ptr(), w, w // 2, w, nb, h,
                                               w, ws.data_ptr(), qout.data_ptr(), flag.data_ptr(),
                                               _device.stream_ptr()))

    for _ in range(max(1, warmup)):
        run_q()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nq = max(3, min(steps, 10))
    e0.record()
    for _ in range(nq):
        run_q()
    e1.record()
    torch.cuda.synchronize()
    per_q = e0.elapsed_time(e1) / nq
    qbytes = (8 * nb + 8 + 2 * nb) * h * w
    res["quality_f64"] = {
        "ms_per_report": round(per_q, 4),
        "flagged": int(flag.item()),
        "roofline": {"bound": "hbm", "achieved": round(qbytes / (per_q * 1e-3) / 1e9, 1),
                     "peak": peak, "unit": "GB/s",
                     "frac": round(qbytes / (per_q * 1e-3) / 1e9 / peak, 4),
                     "algorithmic_bytes_per_report": qbytes,
                     "traffic": ncu_traffic("quality_tile64_kernel_6"),
                     "kernels": "quality_tile64_kernel<6> + quality_edge64_kernel + finish"},
        "api": "wf_quality_scene_f64 / qnr() of float64 planes (was ~87 ms on the per-pair "
               "kernels in round 1)",
    }
    del pan, ms, out, ws
    torch.cuda.empty_cache()
    return {"unit": UNIT, "dtype": "f64 in/out, f64 arithmetic", **res}


def measure_exact(scene, steps, warmup, dist, world, peak):
    """The reference-exact mode on the same f32 scene (fuse(..., exact=True),
    wf_fuse_bands_exact_f32): the reference's own float64 operation sequence
    (fusion.py:148-150, wavelet.py:73-164), bit-identical outputs, one pass
    with no coefficient image. Same algorithmic bytes as the fast kernel."""
    import torch

    from paper_1803_00737_b200 import WaveletKind, _native
    from paper_1803_00737_b200.scene import scene_bytes
    from paper_1803_00737_b200.wavelet import KIND_CODE

    lib = _native.load()
    h, w = scene.shape
    nbytes = scene_bytes(h, w, len(scene.ms))
    ws = torch.empty(1, dtype=torch.float64, device=scene.pan.device)  # one-pass kernels: unused
    ms_p = _native.ptr_array([m.data_ptr() for m in scene.ms])
    out_p = _native.ptr_array([o.data_ptr() for o in scene.out])
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    res = {}
    for kind in (WaveletKind.HAAR, WaveletKind.DAUB4):
        code = KIND_CODE[kind]

        def run():
            _native.check(lib.wf_fuse_bands_exact_f32(code, scene.pan.data_ptr(), w, ms_p, w // 2,
                                                      out_p, w, len(scene.ms), h, w,
                                                      ws.data_ptr(), sp))

        for _ in range(warmup):
            run()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_t = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms_t], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_t = float(t.item())
        per = ms_t / steps
        achieved = nbytes / (per * 1e-3) / 1e9
        sec, h2d, d2h, ok = measure_e2e(scene, kind, max(2, min(steps, 5)), dist,
                                        ref_out=scene.out, exact=True)
        e2e_steps = max(2, min(steps, 5))
        res[kind.value] = {
            "value": round(world * h * w / (per * 1e-3) / 1e6, 3),
            "ms_per_step": round(per, 4),
            "e2e": {"value": round(world * h * w * e2e_steps / sec / 1e6, 3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "wf_fuse_host_f32 with wf_ctx_set_exact (pinned host buffers, "
                           "strips of 1024 rows with halo rows)",
                    "matches_device_result": ok},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "algorithmic_bytes_per_launch": nbytes,
                         "traffic": ncu_traffic("fuse_exact_haar_kernel_float__6__1"
                                                if kind is WaveletKind.HAAR
                                                else "fuse_exact_d4_kernel_float__6__1"),
                         "kernel": ("fuse_exact_haar_kernel<f32,B=6>" if kind is WaveletKind.HAAR
                                    else "fuse_exact_d4_kernel<f32,B=6> (float64 transform "
                                         "order, column-shared)")},
        }
    del ws
    torch.cuda.empty_cache()
    return {"unit": UNIT, "dtype": "f32 in/out, f64 arithmetic in the reference's order",
            "parity": "bit-identical to the reference (tests/test_gpu_parity.py)", **res}


def measure_u8(scene, steps, warmup, dist, world, dev_index, peak):
    """the same scene in the paper's 8 bpp transfer
    representation (uint8 in, quantised uint8 out, float32 arithmetic). A
    step = one launch of the 8 bpp kernel over the whole scene; algorithmic
    bytes (1 + 1.25 B) per PAN px."""
    import torch

    from paper_1803_00737_b200 import WaveletKind, _native
    from paper_1803_00737_b200.fusion import _quantize_dev
    from paper_1803_00737_b200.wavelet import KIND_CODE

    lib = _native.load()
    h, w = scene.shape
    pan = _quantize_dev(scene.pan)
    ms = [_quantize_dev(m) for m in scene.ms]
    out = [torch.empty((h, w), dtype=torch.uint8, device=pan.device) for _ in ms]
    ms_p = _native.ptr_array([m.data_ptr() for m in ms])
    out_p = _native.ptr_array([o.data_ptr() for o in out])
    nbytes = h * w + len(ms) * ((h // 2) * (w // 2) + h * w)
    res = {}
    for kind in (WaveletKind.HAAR, WaveletKind.DAUB4):
        code = KIND_CODE[kind]
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream

        def run():
            _native.check(lib.wf_fuse_bands_u8(code, pan.data_ptr(), w, ms_p, w // 2, out_p, w,
                                               len(ms), h, w, sp))

        for _ in range(warmup):
            run()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_t = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms_t], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_t = float(t.item())
        per = ms_t / steps
        achieved = nbytes / (per * 1e-3) / 1e9
        e2e_steps = max(2, min(steps, 5))
        sec, h2d, d2h, ok = measure_e2e(scene, kind, e2e_steps, dist, pan, ms, [o.clone() for o in out])
        res[kind.value] = {
            "value": round(world * h * w / (per * 1e-3) / 1e6, 3),
            "ms_per_step": round(per, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "algorithmic_bytes_per_launch": nbytes,
                         "traffic": ncu_traffic("fuse_haar_u8_kernel_6" if kind is WaveletKind.HAAR
                                                else "fuse_d4_u8x8_kernel_6"),
                         "kernel": ("fuse_haar_u8_kernel<B=6> (16-bit lanes)"
                                    if kind is WaveletKind.HAAR
                                    else "fuse_d4_u8x8_kernel<B=6, v3> (8 cols/thread, row-pair "
                                         "packed; byte-exact: float32 bytes outside 2^-9 of a "
                                         "rounding boundary, float64 fix-up of the rest)")},
            "e2e": {"value": round(world * h * w * e2e_steps / sec / 1e6, 3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "wf_fuse_host_u8 (C ABI, pinned host buffers, strips of 1024 rows)",
                    "matches_device_result": ok},
        }
    # the round-1 D4 kernel (WF_D4_U8=v2, opt-in): bytes = quantize() of the
    # float32 kernel, <= 1 LSB from the reference -- the price of exactness
    os.environ["WF_D4_U8"] = "v2"
    _native.reload_tuning()
    code = KIND_CODE[WaveletKind.DAUB4]
    sp = torch.cuda.current_stream().cuda_stream

    def run_v2():
        _native.check(lib.wf_fuse_bands_u8(code, pan.data_ptr(), w, ms_p, w // 2, out_p, w,
                                           len(ms), h, w, sp))

    for _ in range(warmup):
        run_v2()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run_v2()
    e1.record()
    torch.cuda.synchronize()
    os.environ.pop("WF_D4_U8")
    _native.reload_tuning()
    per_v2 = e0.elapsed_time(e1) / steps
    res["daub4_v2_not_exact"] = {
        "ms_per_step": round(per_v2, 4),
        "value": round(world * h * w / (per_v2 * 1e-3) / 1e6, 3),
        "roofline_frac": round(nbytes / (per_v2 * 1e-3) / 1e9 / peak, 4),
        "parity": "<= 1 LSB from the reference (~5e-6 of bytes differ); opt-in WF_D4_U8=v2",
    }
    return {"unit": UNIT, "dtype": "u8 in/out, f32 arithmetic (D4: float64 fix-up of values "
                                   "near a rounding boundary)",
            "parity": "byte-identical to the reference worker (tests/test_gpu_quantized.py)",
            **res}


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1803_00737_b200 import WaveletKind
    from paper_1803_00737_b200.scene import DeviceScene, scene_bytes

    dist, local_rank = init_dist(world, local_rank)
    scene = DeviceScene.synthetic(H, W, B, scene=rank)
    torch.cuda.synchronize()
    peak, peak_kind = peaks()
    nbytes = scene_bytes(H, W, B)
    e2e_steps = args.e2e_steps or min(args.steps, 5)
    results = {}
    for kind in (WaveletKind.HAAR, WaveletKind.DAUB4):
        ms, launches, clocks = measure_device(scene, kind, args.steps, args.warmup, dist, world,
                                              local_rank)
        per_launch_ms = ms / max(1, launches)  # one kernel per step
        achieved = nbytes / (per_launch_ms * 1e-3) / 1e9
        sec, h2d, d2h, ok = measure_e2e(scene, kind, e2e_steps, dist)
        results[kind.value] = {
            "value": world * H * W * args.steps / (ms * 1e-3) / 1e6,
            "ms_per_step": ms / args.steps,
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": {
                "bound": "hbm",
                "achieved": round(achieved, 1),
                "peak": peak,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": ncu_traffic(f"fuse_{kind.value}_b6"),
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "frac_of_8tbs_nameplate": round(achieved / 8000.0, 4),
                "algorithmic_bytes_per_launch": nbytes,
                "kernel": ("fuse_haar_kernel<f32,B=6>" if kind is WaveletKind.HAAR
                           else "fuse_d4_tma_kernel<f32,B=6,4 consumer warps>"),
            },
            "e2e": {
                "value": round(world * H * W * e2e_steps / sec / 1e6, 3),
                "unit": UNIT,
                "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "wf_fuse_host_f32 (C ABI, pinned host buffers, strips of 1024 rows)",
                "matches_device_result": ok,
            },
        }
    u8 = measure_u8(scene, args.steps, args.warmup, dist, world, local_rank, peak)
    f64 = measure_f64(scene, args.steps, args.warmup, dist, world, peak)
    exact = measure_exact(scene, args.steps, args.warmup, dist, world, peak)
    quality = measure_quality(scene, args.steps, args.warmup, peak)
    cpu = {}
    if rank == 0 and world == 1 and not args.no_cpu:
        unbind_numa()
        threads = os.cpu_count() or 1
        for kname in ("haar", "daub4"):
            rate, t = cpu_sample(kname, args.cpu_rows, threads)
            cpu[kname] = {
                "value": round(rate, 3), "unit": UNIT, "cores": threads, "kind": "port",
                "sample": (f"first {args.cpu_rows} PAN rows x {W} cols + 6 bands of the scene, "
                           f"{kname}, oracle port of the reference (numpy f64), {t:.2f} s"),
            }
    # BASELINE configs[3] and [4] in the same run (strong scaling over the
    # ranks): the Landsat scene's buffers go back first
    del scene
    torch.cuda.empty_cache()
    c4 = c5 = None
    if not args.no_subconfigs:
        c4 = measure_strips(args, dist, rank, world, local_rank)
        c5 = measure_batch(args, dist, rank, world, local_rank, max(1, args.c5_steps),
                           min(2, max(1, args.warmup)))
    if rank == 0:
        hr = results["haar"]
        line = {
            "metric": METRIC,
            "value": round(hr["value"], 3),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(hr["ms_per_step"], 4),
            "higher_is_better": True,
            "scaling": "weak",
            # the only published number for this path is
            # the paper's HDWT fusion rate (67.5 PAN MPix/s, 16280x14960, 4-node
            # GTX 460 cluster)
            "vs_baseline": round(hr["value"] / PAPER_HDWT_MPIX, 1),
            "baseline_published": {"value": PAPER_HDWT_MPIX, "unit": UNIT,
                                   "source": "BASELINE.md s1 / PAPER.md:153-156 (HDWT, GTX 460 x4)"},
            "dtype": "f32",
            "data": "synthetic (device counter-hash uniform[0,255) f32, Landsat-7-shaped)",
            "config": landsat_config(world),
            "execution": {
                "parallelism": f"scene-sharded replicas x{world} (no collective)",
                "l2": "no flush: 2.24 GB of inputs per step >> 126 MB L2",
                "host_cpus": _BOUND.get("cpus"),
            },
            "gpu_launches": hr["gpu_launches"],
            "clocks": hr["clocks"],
            "roofline": hr["roofline"],
            "e2e": hr["e2e"],
            "cpu_baseline": cpu.get("haar"),
            # both rates -- band-MPix/s = B x scene-MPix/s
            "band_mpix_per_s": round(B * hr["value"], 1),
            "daub4": {
                "value": round(results["daub4"]["value"], 3),
                "vs_baseline": round(results["daub4"]["value"] / PAPER_DDWT_MPIX, 1),
                "ms_per_step": round(results["daub4"]["ms_per_step"], 4),
                "gpu_launches": results["daub4"]["gpu_launches"],
                "clocks": results["daub4"]["clocks"],
                "roofline": results["daub4"]["roofline"],
                "e2e": results["daub4"]["e2e"],
                "cpu_baseline": cpu.get("daub4"),
            },
            # configs[2] at the top level too (the driver parses top-level keys)
            "value_daub4": round(results["daub4"]["value"], 3),
            "ms_per_step_daub4": round(results["daub4"]["ms_per_step"], 4),
            "roofline_frac_daub4": results["daub4"]["roofline"]["frac"],
            "value_strip65536": c4["value"] if c4 else None,
            "value_batch64": c5["value"] if c5 else None,
            "u8_8bpp": u8,
            "f64": f64,
            "exact": exact,
            "quality": quality,
            "strip65536": c4,
            "batch64": c5,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def measure_strips(args, dist, rank, world, local_rank):
    """configs[3]: one N x N D4 scene (1 band) cut into row strips, one per
    rank; each timed step = the halo exchange + the strip kernel. Strong
    scaling: total work fixed. Halo transport: NCCL send/recv ring (default),
    or --halo peer (the neighbours' rows read through CUDA IPC mappings by the
    strip kernel; falls back to NCCL unless every rank can access its ring
    neighbours' memory). Returns the sub-object (rank 0) or None."""
    import torch

    from paper_1803_00737_b200 import WaveletKind, _native, strips, synth
    from paper_1803_00737_b200.scene import scene_bytes

    n = args.strip_size
    r0, r1 = strips.strip_bounds(n, world, rank)
    rows = r1 - r0
    pan = torch.empty((rows, n), device="cuda")
    synth.device_plane(pan, synth.DEFAULT_SEED, synth.plane_id(0, -1), row0=r0)
    ms = torch.empty((rows // 2, n // 2), device="cuda")
    synth.device_plane(ms, synth.DEFAULT_SEED, synth.plane_id(0, 0), row0=r0 // 2)
    out = [torch.empty_like(pan)]
    kind = WaveletKind.DAUB4
    torch.cuda.synchronize()
    if dist:
        dist.barrier()  # all strips exist before neighbours map them
    peer = strips.PeerHalos.try_create(pan, [ms]) if args.halo == "peer" else None
    halo_mode = "peer" if peer is not None else "nccl"

    def step():
        halos = peer if peer is not None else strips.exchange_halos(pan, [ms])
        strips.fuse_strip(kind, pan, [ms], halos, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _native.launch_count()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - n0
    ms_t = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_t = float(t.item())
    peak, peak_kind = peaks()
    strip_bytes = scene_bytes(rows, n, 1)
    per_step = ms_t / args.steps
    achieved = strip_bytes / (per_step * 1e-3) / 1e9
    if dist:
        dist.barrier()  # neighbours finished reading before the mappings go away
    if peer is not None:
        peer.close()
    del pan, ms, out
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    res = {
        "value": round(n * n * args.steps / (ms_t * 1e-3) / 1e6, 3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(per_step, 4),
        "scaling": "strong",
        "workload": (f"C4: one {n}x{n} PAN + 1 MS band f32, D4 periodic wrap, row strips of "
                     f"{rows} rows per rank (BASELINE configs[3])"),
        "halo": ("peer: neighbours' halo rows bulk-copied from their HBM by the strip kernel "
                 "(CUDA IPC), no collective per step") if halo_mode == "peer"
                else "nccl: batched send/recv ring of 2+2 PAN rows + 1 MS row each step",
        "halo_requested": args.halo,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "peak_source": peak_kind, "algorithmic_bytes_per_launch": strip_bytes,
                     "kernel": "fuse_d4_tma_kernel<f32,B=1,4> (strip mode, halo rows)",
                     "note": "per-rank strip bytes / per-step time (halo exchange included)"},
    }
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        crow = 512
        rate, t = cpu_sample_shape("daub4", crow, n, 1, threads)
        res["cpu_baseline"] = {
            "value": round(rate, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"first {crow} PAN rows x {n} cols + 1 band of the C4 scene, D4, oracle "
                       f"port of the reference (numpy f64, exact row strips), {t:.2f} s; a "
                       "per-pixel rate, so no extrapolation to the full scene"),
        }
    return res


def measure_batch(args, dist, rank, world, local_rank, steps, warmup):
    """configs[4]: a batch of Landsat-shaped scenes partitioned by scene over
    the ranks (round-robin, no collective). Per owned scene and per wavelet a
    step runs the fused kernel and the one-pass QNR/ERGAS report on the
    result. Inputs of all owned scenes are device-resident (64 x 2.24 GB fits
    one B200); one output set per rank is reused scene after scene. Returns
    the sub-object (rank 0) or None."""
    import torch

    import paper_1803_00737_b200 as wf
    from paper_1803_00737_b200 import _native, strips, synth
    from paper_1803_00737_b200.scene import DeviceScene

    mine = strips.shard(list(range(args.scenes)), rank, world)
    scenes = []
    out = None
    for s_ in mine:
        sc = DeviceScene.synthetic(H, W, B, seed=synth.DEFAULT_SEED, scene=s_, outputs=out is None)
        if out is None:
            out = sc.out
        else:
            sc.out = out  # share one output set
        scenes.append(sc)
    torch.cuda.synchronize()
    kinds = (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4)
    haar = wf.DwtReplace(wf.WaveletKind.HAAR)
    runs = [(sc, k, sc.launcher(k)) for sc in scenes for k in kinds]
    reports = []

    def step(record):
        # every pass queued back to back; the reports' scalars are read once
        # per step (PendingReport), so the GPU never idles on a per-scene sync.
        # Haar: fusion and report in one pass (fuse_and_qnr_async, row f1);
        # D4: the fused kernel, then the report (qnr_async). (Overlapping a
        # scene's report with the next fusion on two streams measured no
        # gain: the report kernel is persistent, one CTA per SM at the full
        # register file, so the two never share an SM.)
        pending = []
        for sc, kind, run in runs:
            if kind == wf.WaveletKind.HAAR:
                pending.append(wf.fuse_and_qnr_async(sc.pan, sc.ms, haar, out=sc.out)[1])
            else:
                run()
                pending.append(wf.qnr_async(sc.out, sc.ms, sc.pan))
        for p in pending:
            rep = p.result()
            if record:
                reports.append(rep.qnr)

    for _ in range(max(1, warmup)):
        step(False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    n0 = _native.launch_count()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(steps):
            step(True)
        e1.record(stream)
        torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1)
    launches = _native.launch_count() - n0
    if dist:
        t = torch.tensor([ms_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_t = float(t.item())
    del scenes, runs, out
    torch.cuda.empty_cache()
    passes = len(kinds) * args.scenes  # scene-wavelet passes per step, whole job
    if rank != 0:
        return None
    res = {
        "value": round(passes * H * W * steps / (ms_t * 1e-3) / 1e6, 3),
        "unit": "scene-MPix/s (fused + QNR report per scene and wavelet)",
        "n_gpus": world,
        "steps": steps,
        "warmup": max(1, warmup),
        "ms_per_step": round(ms_t / steps, 3),
        "scaling": "strong",
        "workload": (f"C5: {args.scenes} Landsat-shaped scenes x (Haar, D4), each fused and "
                     "scored (QNR/ERGAS) on the GPU (BASELINE configs[4]); Haar in one pass "
                     "(fuse_and_qnr_async), D4 as fusion then report in the same call"),
        "global_batch": args.scenes,
        "parallelism": f"scene-sharded x{world} (round-robin, no collective)",
        "scenes_per_rank": len(mine),
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "qnr_sample": round(float(sum(reports) / max(1, len(reports))), 6),
    }
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        crow = 512
        rate, t = cpu_sample_shape("haar", crow, W, B, threads, with_qnr=True)
        res["cpu_baseline"] = {
            "value": round(rate, 4), "unit": res["unit"], "cores": threads, "kind": "port",
            "sample": (f"first {crow} PAN rows x {W} cols + {B} bands of one scene, Haar "
                       f"fused (oracle port, {threads} threads) and scored (oracle qnr, one "
                       f"thread), {t:.1f} s; per-pixel rate of one scene-wavelet pass"),
        }
    return res


def _standalone_line(sub, args):
    line = {"metric": METRIC, "higher_is_better": True, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device counter-hash uniform[0,255) f32)"}
    line.update({k: v for k, v in sub.items() if k != "workload"})
    line["config"] = {"workload": sub["workload"], "global_batch": sub.get("global_batch", 1),
                      "parallelism": sub.get("parallelism", f"row strips x{sub['n_gpus']}"),
                      "l2": "no flush: inputs >> 126 MB L2"}
    return line


def run_strips(args, rank, world, local_rank):
    dist, local_rank = init_dist(world, local_rank)
    sub = measure_strips(args, dist, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(_standalone_line(sub, args)), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_batch(args, rank, world, local_rank):
    dist, local_rank = init_dist(world, local_rank)
    sub = measure_batch(args, dist, rank, world, local_rank, args.steps, args.warmup)
    if rank == 0:
        print(json.dumps(_standalone_line(sub, args)), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_plumbing(args, rank, world):
    """CPU-only check of the multi-process plumbing (spawn, rendezvous, barrier,
    max-over-ranks timing, rank-0 JSON line) with gloo: no GPU work, so the
    CPU test suite can prove `bench.py --gpus N` really starts N ranks."""
    import numpy as np
    import torch
    import torch.distributed as td

    if world > 1:
        td.init_process_group("gloo")
    a = np.random.default_rng(rank).random((256, 256))
    for _ in range(args.warmup):
        a = a @ a.T / 256.0
    if world > 1:
        td.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a = a @ a.T / 256.0
    sec = time.perf_counter() - t0
    ranks = torch.tensor([float(rank)])
    t = torch.tensor([sec])
    if world > 1:
        td.all_reduce(t, op=td.ReduceOp.MAX)
        td.all_reduce(ranks, op=td.ReduceOp.SUM)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "workload": "plumbing (no GPU work)", "n_gpus": world,
                          "world_size": world, "rank_sum": int(ranks.item()),
                          "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(1e3 * float(t.item()) / max(1, args.steps), 4)}),
              flush=True)
    if world > 1:
        td.barrier()
        td.destroy_process_group()


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun's environment: start N ranks, one
    process per GPU, through torch.distributed.run on 127.0.0.1 (the same
    launch the driver uses), and return their exit status. Rank 0 prints the
    JSON line."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.workload == "plumbing":
        run_plumbing(args, rank, world)
        return
    if args.workload == "strip65536":
        run_strips(args, rank, world, local_rank)
        return
    if args.workload == "batch64":
        run_batch(args, rank, world, local_rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
