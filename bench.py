#!/usr/bin/env python3
"""bench.py — frames/s of the change-based scene-labeling net on B200.

Workload (BASELINE.json configs[1]): the paper's scene-labeling net
(make_seg7_spec layer list, io.cpp:568-617, derived dims) at 640x480, weights
fill_random_weights(seed 1), tau = 0.05 on every conv layer, S independent
camera streams per GPU; stream g (global id) is gen_synthetic{seed 1000+g,
n_objects, object_size, velocity} (io.cpp:499-552). A "step" = one frame of
every stream on this GPU through the whole per-frame hot path
(detect -> dilate/compact -> gather+tcgen05 GEMM+scatter -> CB max-pool, 18
kernels in one CUDA graph). The bootstrap frame is excluded.

  value : whole-job frames/s, frames already resident in HBM (zero-copy ingest)
  e2e   : same metric through the public C ABI with HOST frames (pinned), the
          H2D copy of each step's frames and the D2H copy of each step's result
          (last node's retained output, all streams) inside the timed region
  roofline : dominant kernel, algorithmic bytes/flops per launch / CUDA-event
          duration (instrumented pass on the same sequence)
  cpu_baseline : the unmodified reference (oracle/_ref/ref_bench, one CBNetwork
          per host thread), rank 0 at N=1, bounded sample

Multi-GPU: one process per GPU (torchrun), streams sharded by rank, no data-path
collective; barrier + max-over-ranks of the device time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s per B200 vs changed-pixel % (scene-labeling net); % HBM/TC roofline"
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


# BASELINE.json configs this bench runs: configs[1] (the metric's workload, the
# default; weak scaling, streams per GPU) and configs[4] (64 x 1080p streams
# sharded over the ranks: strong scaling, the driver's SCALE run with --config cfg5)
CONFIGS = {
    "cfg2": dict(height=480, width=640, streams=64, groups=4, ring=16, objects=6, object_size=40, velocity=4,
                 scaling="weak", sweep_steps=6),
    "cfg5": dict(height=1080, width=1920, streams=64, groups=4, ring=4, objects=12, object_size=80, velocity=4,
                 scaling="strong", sweep_steps=0),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS),
                    help="cfg2: scene-labeling net 640x480, 64 streams per GPU (weak); cfg5: 64 x 1920x1080 "
                         "streams in total, sharded over the GPUs (strong)")
    ap.add_argument("--streams", type=int, default=None,
                    help="camera streams per GPU (cfg2) / in total over all GPUs (cfg5)")
    ap.add_argument("--groups", type=int, default=None,
                    help="stream groups per GPU, each its own stream set on its own CUDA stream (overlap)")
    ap.add_argument("--ring", type=int, default=None, help="distinct frames per stream (ping-pong playback)")
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--objects", type=int, default=None)
    ap.add_argument("--object-size", type=int, default=None)
    ap.add_argument("--velocity", type=int, default=None)
    ap.add_argument("--noise", type=float, default=0.0)
    ap.add_argument("--tau", type=float, default=0.05)
    ap.add_argument("--profile-steps", type=int, default=5, help="instrumented steps for the roofline")
    ap.add_argument("--dense-steps", type=int, default=5, help="steps of the dense (full-update) path")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU-baseline work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ingest", choices=["u8", "f32"], default="u8",
                    help="device-resident frame format of the value / roofline / dense / sweep passes: the 8-bit "
                         "PNM payload (cbg_net_forward_u8) or its fp32 conversion (cbg_net_forward)")
    ap.add_argument("--sweep-steps", type=int, default=None,
                    help="timed steps per point of the change-rate sweep (0 disables the sweep)")
    ap.add_argument("--persistent-sms", type=int, default=-1,
                    help="SMs each stream group's persistent GEMM / conv kernels spread over (0 = all; default "
                         "-1: a third of the SMs with 3 or more groups, else SMs / groups)")
    ap.add_argument("--cpu-one-core-budget", type=float, default=8.0,
                    help="seconds of the 1-thread, 1-stream CPU reference sample (0 disables)")
    a = ap.parse_args()
    for k, v in CONFIGS[a.config].items():
        if getattr(a, k, None) is None:
            setattr(a, k, v)
    return a


def local_streams(a, rank, world):
    """(shard, stream count on this rank, stream groups) of the configured workload"""
    from paper_1808_05488_b200.sharding import shard_streams, weak_shard
    shard = weak_shard(a.streams, rank, world) if a.scaling == "weak" else shard_streams(a.streams, rank, world)
    S = shard.count
    G = max(g for g in range(1, a.groups + 1) if S % g == 0)
    return shard, S, G


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config_dict(a, world):
    total = a.streams * world if a.scaling == "weak" else a.streams
    per = f"{a.streams} streams/GPU" if a.scaling == "weak" else f"{a.streams} streams sharded over {world} GPU(s)"
    return {"workload": f"{a.config}: scene-labeling net (seg7 layers, derived dims) {a.width}x{a.height}, "
                        f"{per}, gen_synthetic {a.objects}x{a.object_size}px objects "
                        f"v={a.velocity} noise={a.noise}, tau={a.tau}",
            "baseline_config": a.config, "height": a.height, "width": a.width,
            "streams_per_gpu": a.streams if a.scaling == "weak" else -(-a.streams // world),
            "total_streams": total, "stream_groups": a.groups, "frame_ring": a.ring,
            "objects": a.objects, "object_size": a.object_size,
            "velocity": a.velocity, "noise_std": a.noise, "tau": a.tau,
            "frames": "gen_synthetic quantized to 8-bit PNM payloads; fp32 arms see load_pnm's byte/255.0f",
            "ingest": (f"value/roofline/dense/sweep: device-resident {getattr(a, 'ingest', 'u8')} frames "
                       "(u8 = the PNM payload through cbg_net_forward_u8, f32 = its byte/255.0f through "
                       "cbg_net_forward)"),
            "parallelism": f"streams sharded over {world} GPU(s), no collective",
            "persistent_sms_per_group": getattr(a, "psms", None),
            "l2": "inputs larger than L2 (frame ring + per-stream state >> 126 MB)"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref/ref_bench = the unmodified reference build)
# ---------------------------------------------------------------------------
def run_ref_bench(a, threads, frames, budget, streams=None):
    if not os.path.exists(REF_BENCH):
        return None
    streams = streams or threads
    cmd = [REF_BENCH, "--height", str(a.height), "--width", str(a.width), "--streams", str(streams),
           "--threads", str(threads), "--frames", str(frames), "--objects", str(a.objects),
           "--object-size", str(a.object_size), "--velocity", str(a.velocity), "--noise", str(a.noise),
           "--tau", str(a.tau), "--time-budget", str(budget), "--pnm8"]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def reference_arm(a, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    base = {"metric": METRIC, "unit": "frames/s", "impl": "reference", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (gen_synthetic, seeded)", "config": config_dict(a, world)}
    if not os.path.exists(REF_BENCH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    # each step = one frame of every host-thread stream; bootstrap excluded
    r = run_ref_bench(a, threads, max(1, a.steps), budget=max(10.0, a.cpu_budget * 3))
    sample = (f"{r['frames']} post-bootstrap frames over {r['streams']} streams ({threads} threads), "
              f"L1 change {100 * r['l1_change_frac']:.2f}%")
    base.update({"value": r["fps"], "ms_per_step": 1000.0 * r["seconds"] / max(1, r["frames"]) * threads,
                 "cpu_baseline": {"value": r["fps"], "unit": "frames/s", "cores": threads, "kind": "reference",
                                  "sample": sample},
                 "e2e": {"value": r["fps"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(base))


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """Polls NVML (SM clock, max clock, clock-event reasons) every ~1 ms in a
    thread while the timed region runs (nvidia-smi -lms cannot resolve a
    region of a few tens of ms)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, local_rank):
        self.local = local_rank
        self.rows = []
        self.stop = threading.Event()
        self.handle = None
        self.max_mhz = None

    def _open(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.local)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.local)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)

    def _poll(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM),
                                  get_reasons(self.handle)))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        try:
            self._open()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.handle = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.handle is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, r in self.rows for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, ~1 ms polling in the timed region"}


# change-rate sweep points (objects, object size) -> L1-output change of
# ~0.1 / 0.4 / 1.2 / 3 / 6 / 15 / 28 % at 640x480 (gen_synthetic, v=4), plus
# "random": every frame i.i.d. uniform noise, so ~100% of pixels change on
# every layer (the change-based path's worst case, compared with the dense path)
SWEEP = [(1, 8), (2, 16), (3, 32), (6, 40), (10, 48), (24, 64), (60, 96), "random"]


# ---------------------------------------------------------------------------
# algorithmic work per kernel launch
# ---------------------------------------------------------------------------
def receptive_union(out_mask, hin, win, kh, kw, st, pad):
    """U: input pixels inside the receptive field of any marked output pixel
    (the distinct pixels a gather has to read once)."""
    import numpy as np
    ho, wo = out_mask.shape
    m = np.zeros((hin, win), bool)

    def rng(k, n_out, n_in):  # output range whose tap k lands inside the input
        o0 = max(0, -(-(pad - k) // st))
        o1 = min(n_out, (n_in - 1 + pad - k) // st + 1)
        return o0, o1
    for kj in range(kh):
        j0, j1 = rng(kj, ho, hin)
        if j0 >= j1:
            continue
        for ki in range(kw):
            i0, i1 = rng(ki, wo, win)
            if i0 >= i1:
                continue
            m[j0 * st - pad + kj:(j1 - 1) * st - pad + kj + 1:st,
              i0 * st - pad + ki:(i1 - 1) * st - pad + ki + 1:st] |= out_mask[j0:j1, i0:i1]
    return int(m.sum())


def kernel_work(kn, nd, n_out, n_det, n_up, u_ratio, ingest, pool_of=None, n_pool=None):
    """Algorithmic (bytes, flops) of one launch of kernel kn of node nd, summed
    over the streams. n_out / n_det / n_up: per-stream changed output pixels,
    detected input pixels (before dilation) and the producer's changed pixels;
    u_ratio: U / n_out of the node's gather (receptive_union, sampled)."""
    cin, hin, win = nd["in"]
    cout, hout, wout = nd["out"]
    k2 = nd["k"] ** 2
    b = f = 0.0
    for s in range(len(n_out)):
        no, nd_ = float(n_out[s]), float(n_det[s]) if n_det is not None else 0.0
        if kn == "detect":
            if n_up is None:  # first layer, dense over the frame
                if ingest == "u8":  # 8-bit frame + 8-bit state shadow read; fp32 state + shadow written
                    b += 2.0 * cin * hin * win + 5.0 * cin * nd_
                else:               # fp32 frame + fp32 state read, state written
                    b += 8.0 * cin * hin * win + 4.0 * cin * nd_
            else:             # x and state at the producer's update set, state (+ pre-split copy) written
                b += 8.0 * cin * float(n_up[s]) + 4.0 * cin * nd_ * (2 if nd["presplit"] else 1)
            b += hin * win / 8.0  # bitmap
        elif kn == "dilcomp":
            b += hin * win / 8.0 + hout * wout / 8.0 + 4.0 * no
            if pool_of is not None:
                b += pool_of["out"][1] * pool_of["out"][2] / 8.0 + 4.0 * float(n_pool[s])
        elif kn == "gemm":
            f += nd["ops_pp"] * no
            b += 4.0 * cin * u_ratio * no + 4.0 * cout * no
        elif kn == "pool":
            b += 4.0 * cin * 4 * no + 4.0 * cin * no
        elif kn == "join":
            b += 4.0 * cout * (nd["n_in"] + 1) * no
    if kn == "gemm":
        b += 4.0 * cout * cin * k2  # weights (fp16 hi + lo images, or fp32) once per launch
    return b, f


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.impl == "reference":
        reference_arm(a, rank, world)
        return

    import numpy as np
    import torch

    # BENCH_DEVICE_MOD / BENCH_DIST_BACKEND only exist to exercise the N>1 code
    # path on a one-GPU box (ranks share the device over gloo); the driver's runs
    # use one GPU per rank over NCCL.
    local = local % int(os.environ.get("BENCH_DEVICE_MOD", "1000000"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1808_05488_b200 import cbi
    from paper_1808_05488_b200.sharding import max_over_ranks as _max_over_ranks

    peaks = {"hbm_gbs": 6538.6, "bf16_tflops": 1661.9, "bf16_tflops_sustained": 1399.9, "sm_max_mhz": 1965.0,
             "source": "fallback (B200_PROFILING.md)"}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        with open(pk_path) as fh:
            peaks.update(json.load(fh))
        peaks["source"] = "measured (MEASURED_PEAKS.json)"
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count

    shard, S, G = local_streams(a, rank, world)
    H, W = a.height, a.width
    Sg = S // G
    ctxs = [cbi.Context(local) for _ in range(G)]
    ctx = ctxs[0]
    # the groups' GEMMs share the GPU side by side instead of each taking every
    # SM (measured: 57.5k frames/s with all 148 SMs per GEMM, 60-62k with 50-56)
    psms = a.persistent_sms if a.persistent_sms >= 0 else (-(-n_sm // 3) if G >= 3 else -(-n_sm // G))
    for c in ctxs:
        c.set_persistent_sms(psms)
    a.psms = psms
    spec = cbi.make_seg_spec(1, H, W)
    taus = [a.tau] * 5
    L = max(3, a.ring)
    # frame ring [L][S][H][W][C], 8-bit PNM payloads (what a camera or `cbi run`'s
    # PNM sequence delivers: load_pnm, io.cpp:349-399), pinned on the host and
    # resident in HBM; played ping-pong (1..L-1, L-2..2, ...) so motion stays
    # continuous for any step count. The fp32 arms see load_pnm's byte / 255.0f
    # of the same bytes (IEEE division), so every arm runs one workload.
    host8 = torch.empty((L, S, H, W, 3), dtype=torch.uint8, pin_memory=True)
    h8np = host8.numpy()
    from concurrent.futures import ThreadPoolExecutor

    def _gen(s_):
        h8np[:, s_] = cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(
            H, W, 3, L, a.objects, a.object_size, a.velocity, a.velocity, a.noise, shard.seed(s_))))
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        list(pool.map(_gen, range(S)))
    dev8 = host8.to(f"cuda:{local}")
    u8_in = a.ingest == "u8"
    dev = None
    if not u8_in:  # [L][S][C][H][W] fp32 = byte / 255.0f
        dev = (dev8.permute(0, 1, 4, 2, 3).float() / 255.0).contiguous()
    torch.cuda.synchronize()

    def feed(net_, t, g=None):
        """one frame of the device-resident workload (all streams of group g, or of the whole set)"""
        if u8_in:
            net_.enqueue_device_u8((dev8[t] if g is None else dev8[t, g * Sg]).data_ptr())
        else:
            net_.enqueue_device((dev[t] if g is None else dev[t, g * Sg]).data_ptr())
    order = list(range(1, L)) + list(range(L - 2, 1, -1))

    def frame_at(k):  # frame index of post-bootstrap step k
        return order[k % len(order)]

    frame_bytes = S * 3 * H * W * 4
    frame8_bytes = S * 3 * H * W

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        return _max_over_ranks(x, device=f"cuda:{local}")

    exts = [torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", local)) for c in ctxs]
    # the contexts' copy-out streams (copy_output_detached) end inside the timed region too
    exts += [torch.cuda.ExternalStream(c.copy_stream, device=torch.device("cuda", local)) for c in ctxs]
    ext = exts[0]
    nets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
    net = nets[0]
    n_slots, node_slot = net.count_layout()
    det_slot = net.detect_slots()
    nodes = net.nodes()
    counts_pinned = torch.empty((G, a.steps + 1, Sg, n_slots), dtype=torch.int32, pin_memory=True)

    def timed_region(step_fn, steps, finish=None):
        """device time of `steps` calls of step_fn(k) across all groups (CUDA
        events); finish() runs on the host before the end event is recorded"""
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(ext)
        for e in exts[1:]:
            e.wait_event(t0)
        for k in range(steps):
            step_fn(k)
        if finish is not None:
            finish()
        for e in exts[1:]:
            ev = torch.cuda.Event()
            ev.record(e)
            ext.wait_event(ev)
        t1.record(ext)
        # wait with the GIL released (the NVML clock poller runs meanwhile)
        while not t1.query():
            time.sleep(0.0002)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    def change_of(cnt):
        """cnt [..., S, slot] -> (L1-output fraction, L1 detected-input fraction, per-layer fractions)"""
        l1_px = nodes[0].out_shape[1] * nodes[0].out_shape[2]
        in_px = nodes[0].in_shape[1] * nodes[0].in_shape[2]
        per = {n.name: float(cnt[..., node_slot[i]].mean()) / (n.out_shape[1] * n.out_shape[2])
               for i, n in enumerate(nodes)}
        return (float(cnt[..., node_slot[0]].mean()) / l1_px, float(cnt[..., det_slot[0]].mean()) / in_px, per)

    # ---- value: frames resident in HBM ---------------------------------------
    for g in range(G):
        feed(nets[g], 0, g)  # bootstrap (untimed)
    for k in range(a.warmup):
        for g in range(G):
            feed(nets[g], frame_at(k), g)
    for c in ctxs:
        c.synchronize()
    barrier()
    base_k = a.warmup

    def value_step(k):
        for g in range(G):
            feed(nets[g], frame_at(base_k + k), g)
            nets[g].copy_counts_async(counts_pinned[g, k].data_ptr())

    with ClockSampler(local) as clocks:
        ms = max_over_ranks(timed_region(value_step, a.steps))
    barrier()
    launches = net.last_launches() * G
    cnt = np.concatenate([counts_pinned[g, :a.steps].numpy() for g in range(G)], axis=1)  # [step][S][slot]
    l1_frac, l1_det_frac, per_layer = change_of(cnt)
    total_streams = S * world if a.scaling == "weak" else a.streams
    value = total_streams * a.steps / (ms / 1000.0)
    next_k = base_k + a.steps
    labels = net.kernel_labels()

    # ---- roofline: instrumented pass (per-kernel CUDA events) -----------------
    # one stream set holding all S streams (the launch shape of the ncu capture
    # in profiles/), eager launches with an event pair around every kernel
    pctx = cbi.Context(local)  # every SM: the kernels are timed alone (the ncu capture's launch shape)
    pnet = cbi.convert_to_cb(spec, taus, n_streams=S, ctx=pctx)
    feed(pnet, 0)
    for k in range(2):
        feed(pnet, frame_at(next_k + k))
    pctx.synchronize()
    pnet.set_kernel_timing(True)
    layer = {ld.name: ld for ld in spec.layers}
    desc = []
    for i, n in enumerate(nodes):
        ld = layer.get(n.name)
        k = ld.conv.kernel_h if (ld is not None and n.kind == cbi.LayerKind.Conv) else 1
        desc.append({"in": tuple(n.in_shape), "out": tuple(n.out_shape), "k": k, "ops_pp": int(n.ops_per_pixel),
                     "presplit": n.kind == cbi.LayerKind.Conv and k > 1 and n.out_shape[0] > 16
                     and bool(n.inputs) and n.inputs[0] >= 0,
                     "n_in": len(n.inputs), "conv": ld.conv if n.kind == cbi.LayerKind.Conv else None})
    # pools whose map and list come from their producer's compaction (no own dilcomp launch)
    fused_pool = {n.inputs[0]: i for i, n in enumerate(nodes)
                  if n.kind == cbi.LayerKind.Pool and f"{n.name}.dilcomp" not in labels}
    work = {}
    prof_counts = torch.empty((S, n_slots), dtype=torch.int32, pin_memory=True)
    u_ratio = {}
    for k in range(a.profile_steps):
        feed(pnet, frame_at(next_k + 2 + k))
        pnet.copy_counts_async(prof_counts.data_ptr())
        pctx.synchronize()
        c = prof_counts.numpy().T  # [slot][S]
        if k == a.profile_steps - 1 or not u_ratio:
            # U / n_out of each conv's gather on a sample of streams of this frame
            for i, n in enumerate(nodes):
                cv = desc[i]["conv"]
                if cv is None:
                    continue
                num = den = 0
                for sidx in range(min(S, 8)):
                    m, _ = pnet.node_changes(i, sidx)
                    num += receptive_union(m.astype(bool), n.in_shape[1], n.in_shape[2], cv.kernel_h, cv.kernel_w,
                                           cv.stride, cv.padding)
                    den += int(m.sum())
                u_ratio[i] = num / den if den else 1.0
        for i, n in enumerate(nodes):
            src = n.inputs[0] if n.inputs else -1
            n_out = c[node_slot[i]]
            n_det = c[det_slot[i]] if det_slot[i] >= 0 else None
            n_up = c[node_slot[src]] if src >= 0 else None
            kinds = {cbi.LayerKind.Conv: ("detect", "dilcomp", "gemm"), cbi.LayerKind.Pool: ("dilcomp", "pool")}
            for kern in kinds.get(n.kind, ("dilcomp", "join")):
                pc = fused_pool.get(i)
                bb, ff = kernel_work(kern, desc[i], n_out, n_det, n_up, u_ratio.get(i, 1.0), a.ingest,
                                     desc[pc] if (kern == "dilcomp" and pc is not None) else None,
                                     c[node_slot[pc]] if pc is not None else None)
                wsum = work.setdefault(f"{n.name}.{kern}", [0.0, 0.0, 0])
                wsum[0] += bb
                wsum[1] += ff
                wsum[2] += 1
    rep = pnet.timing_report()
    pnet.set_kernel_timing(False)
    del pnet
    traffic, ncu_us = {}, {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("streams") == S and tj.get("height") == H and tj.get("width") == W:
            traffic = tj.get("dram_bytes_per_launch", {})
            ncu_us = tj.get("duration_us", {})
    hbm = peaks["hbm_gbs"] * 1e9
    # the tcgen05 GEMMs run kind::f16 (3xFP16 split, default) or kind::tf32
    # (CBG_GEMM_PREC=tf32); the tensor peak is that kind's dense rate: the
    # measured bf16 (= fp16) rate, or half of it for tf32
    f16_gemm = os.environ.get("CBG_GEMM_PREC", "f16") != "tf32"
    tc = peaks["bf16_tflops"] * 1e12 / (1 if f16_gemm else 2)
    # the bit-exact CUDA-core convs (Cout <= 16) issue one non-fused fp32 mul
    # and one add per MAC: 1 flop per lane per clock on 128 lanes per SM
    fp32 = n_sm * 128 * peaks["sm_max_mhz"] * 1e6
    exact = {n.name for n in nodes if n.kind == cbi.LayerKind.Conv and n.out_shape[0] <= 16}
    kernels = []
    for label, (tot_ms, nl) in rep["kernels"].items():
        bb, ff, nw = work.get(label, [0.0, 0.0, 1])
        bb, ff = bb / max(1, nw), ff / max(1, nw)  # per launch
        t = tot_ms / 1000.0 / max(1, nl)
        fpk = fp32 if label.split(".")[0] in exact else tc
        t_roof = max(bb / hbm, ff / fpk)
        bound = ("fp32" if fpk == fp32 else "tensor") if ff / fpk > bb / hbm else "hbm"
        kk = {"kernel": label, "ms_per_launch": 1000.0 * t, "share": 0.0, "bytes_per_launch": bb,
              "flops_per_launch": ff, "roofline_frac": (t_roof / t) if t > 0 else None, "bound": bound}
        if label in traffic and ncu_us.get(label):
            kk["ncu_dram_bytes"] = traffic[label]
            kk["ncu_us"] = ncu_us[label]
            kk["ncu_dram_frac"] = traffic[label] / (ncu_us[label] * 1e-6) / hbm
        kernels.append(kk)
    tot = sum(k["ms_per_launch"] for k in kernels) or 1.0
    for k in kernels:
        k["share"] = k["ms_per_launch"] / tot
    kernels.sort(key=lambda k: -k["ms_per_launch"])
    dom = kernels[0]
    if dom["bound"] in ("tensor", "fp32"):
        pk = tc if dom["bound"] == "tensor" else fp32
        achieved = dom["flops_per_launch"] / (dom["ms_per_launch"] / 1000.0) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk / 1e12, "unit": "TFLOP/s",
                "frac": achieved / (pk / 1e12)}
        if dom["bound"] == "tensor":
            # the split-fp32 product issues 3 MMAs per useful MAC: the tensor
            # pipe's share is 3x the useful fraction (attainable useful frac <= 1/3)
            roof["tensor_issue_frac"] = 3 * achieved / (pk / 1e12)
            roof["peak_note"] = (("fp16 dense = measured bf16 rate (burst)" if f16_gemm else "tf32 dense = measured "
                                  "bf16 / 2") + "; useful fp32-accurate flops (2*Cout*Cin*k^2 per changed px), "
                                 "3 MMAs per useful MAC")
    else:
        achieved = dom["bytes_per_launch"] / (dom["ms_per_launch"] / 1000.0) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    roof.update({"kernel": dom["kernel"], "traffic": traffic.get(dom["kernel"]),
                 "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, profiles/ncu_traffic.json",
                 "launch_streams": S, "peak_source": peaks["source"],
                 "work_model": ("algorithmic bytes/flops per launch from the device counts (DESIGN.md §3): detect "
                                "2*Cin B/px of 8-bit frame+shadow (u8) or 8*Cin (f32) + state writes at detected px; "
                                "detect_list 8*Cin per producer-changed px + 4*Cin per detected px (x2 with the "
                                "pre-split copy); dilcomp bitmaps in+out + 4 B per listed px (+ a fused pool's); "
                                "gemm 4*Cin*U + 4*Cout*n_out + weights (U = receptive-field union, sampled on "
                                "8 streams); pool 4*C*(4+1) per px"),
                 "peaks": {"hbm_gbs": peaks["hbm_gbs"], "tensor_tflops": tc / 1e12, "fp32_tflops": fp32 / 1e12},
                 "step_roofline_frac": (sum(max(k["bytes_per_launch"] / hbm, k["flops_per_launch"] /
                                                (fp32 if k["kernel"].split(".")[0] in exact else tc))
                                            for k in kernels) / (tot / 1000.0)),
                 "top_kernels": kernels[:8],
                 "all_kernels": {k["kernel"]: {"us": round(1000 * k["ms_per_launch"], 1),
                                               "frac": round(k["roofline_frac"] or 0.0, 3), "bound": k["bound"],
                                               **({"ncu_us": k["ncu_us"], "ncu_dram_frac": round(k["ncu_dram_frac"], 3)}
                                                  if "ncu_us" in k else {})}
                                 for k in kernels},
                 "u_ratio": {nodes[i].name: round(v, 3) for i, v in u_ratio.items()}})

    # ---- dense path (same kernels, every frame a full update) -------------------
    dense_fps = None
    if a.dense_steps > 0:
        # its best setting: every group's GEMMs on every SM (the full update is
        # tensor-bound; the SM share only helps the change-based path)
        dctxs = [cbi.Context(local) for _ in range(G)]
        dexts = [torch.cuda.ExternalStream(c.stream, device=torch.device("cuda", local)) for c in dctxs]
        dnets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=dctxs[g]) for g in range(G)]
        for g in range(G):
            dnets[g].set_dense(True)
            feed(dnets[g], 0, g)
            feed(dnets[g], 1, g)
        for c in dctxs:
            c.synchronize()

        def dense_step(k):
            for g in range(G):
                feed(dnets[g], frame_at(k), g)

        saved = list(exts)
        exts[:] = dexts
        ext = dexts[0]
        try:
            dms = max_over_ranks(timed_region(dense_step, a.dense_steps))
        finally:
            exts[:] = saved
            ext = exts[0]
        dense_fps = total_streams * a.dense_steps / (dms / 1000.0)
        del dnets

    # ---- change-rate sweep: frames/s vs changed-pixel % (the metric's x-axis) ---
    sweep = []
    if a.sweep_steps > 0:
        R = 6
        sorder = list(range(1, R)) + list(range(R - 2, 1, -1))
        sw_counts = torch.empty((G, Sg, n_slots), dtype=torch.int32, pin_memory=True)
        for pt in SWEEP:
            if pt == "random":
                gen = torch.Generator(device=f"cuda:{local}").manual_seed(4242 + rank)
                sdev8 = torch.randint(0, 256, (R, S, H, W, 3), generator=gen, device=f"cuda:{local}",
                                      dtype=torch.uint8)
            else:
                ob, sz = pt
                sh = torch.empty((R, S, H, W, 3), dtype=torch.uint8, pin_memory=True)
                shn = sh.numpy()

                def _gen_s(s_, ob=ob, sz=sz, shn=shn):
                    shn[:, s_] = cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(
                        H, W, 3, R, ob, sz, a.velocity, a.velocity, a.noise, shard.seed(s_))))
                with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
                    list(pool.map(_gen_s, range(S)))
                sdev8 = sh.to(f"cuda:{local}")
            sdev = sdev8 if u8_in else (sdev8.permute(0, 1, 4, 2, 3).float() / 255.0).contiguous()

            def sfeed(net_, t, g, sdev=sdev):
                if u8_in:
                    net_.enqueue_device_u8(sdev[t, g * Sg].data_ptr())
                else:
                    net_.enqueue_device(sdev[t, g * Sg].data_ptr())
            snets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
            for g in range(G):
                sfeed(snets[g], 0, g)
            for k in range(3):
                for g in range(G):
                    sfeed(snets[g], sorder[k % len(sorder)], g)
            for c in ctxs:
                c.synchronize()
            barrier()

            def sweep_step(k, snets=snets, sfeed=sfeed):
                for g in range(G):
                    sfeed(snets[g], sorder[(3 + k) % len(sorder)], g)

            sms = max_over_ranks(timed_region(sweep_step, a.sweep_steps))
            for g in range(G):
                snets[g].copy_counts_async(sw_counts[g].data_ptr())
            for c in ctxs:
                c.synchronize()
            sc = np.concatenate([sw_counts[g].numpy() for g in range(G)], axis=0)  # [S][slot]
            fr, dfr, per = change_of(sc)
            fps = total_streams * a.sweep_steps / (sms / 1000.0)
            sweep.append({"synthetic": ("uniform noise every frame" if pt == "random"
                                        else f"{pt[0]} objects x {pt[1]} px"),
                          "l1_changed_pct": 100.0 * fr, "input_detected_pct": 100.0 * dfr,
                          "per_layer_changed_pct": {k_: round(100.0 * v_, 3) for k_, v_ in per.items()},
                          "frames_per_s": fps,
                          "speedup_vs_dense": (fps / dense_fps) if dense_fps else None})
            del snets, sdev, sdev8
        torch.cuda.empty_cache()
    crossover = None
    if dense_fps and sweep:
        import math
        pts = sorted((p["l1_changed_pct"], p["frames_per_s"] / dense_fps) for p in sweep)
        for (x0, r0), (x1, r1) in zip(pts, pts[1:]):
            if r0 >= 1.0 > r1:  # linear in log(change) between the bracketing points
                f = (r0 - 1.0) / (r0 - r1)
                crossover = math.exp(math.log(max(x0, 1e-6)) + f * (math.log(x1) - math.log(max(x0, 1e-6))))
                break

    # ---- e2e: host frames through the C ABI, H2D + D2H in the timed region -------
    # headline: 8-bit PNM payloads (cbg_net_forward_u8, load_pnm's conversion on
    # the device); also the fp32 Tensor3 API (cbg_net_forward) with host frames
    e2e = e2e_f32 = e2e_full = None
    if not a.no_e2e:
        hnp = None
        if a.config == "cfg2":  # host fp32 frames (4x the bytes) for the Tensor3 arm
            hnp = torch.empty((L, S, 3, H, W), dtype=torch.float32, pin_memory=True).numpy()
            for t in range(L):
                hnp[t] = cbi.from_pnm8(h8np[t])

        def run_e2e(u8, delta):
            """host frames in (H2D inside), the step's result out: delta = this
            frame's changed pixels of the last node + their output vectors, written
            into pinned host memory by the copy-out kernel and scattered into a
            persistent host mirror of the full output (step k applied while steps
            k+1..k+LAG run, one host thread per stream group); else the whole
            output (copy_output_detached)"""
            LAG = 3
            enets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
            out_bytes = enets[0].output_bytes(-1)
            if delta:
                dbufs = [[cbi.HostBuffer(enets[g].output_delta_bytes(-1)) for _ in range(LAG + 1)] for g in range(G)]
                mirrors = [np.zeros(out_bytes // 4, np.float32) for _ in range(G)]
                appl = ThreadPoolExecutor(max_workers=G)
                dbytes, dma = [], []
            else:
                out_host = [torch.empty(out_bytes // 4, dtype=torch.float32, pin_memory=True) for _ in range(G)]

            def put(g, k):
                if u8:
                    enets[g].enqueue_u8(h8np[k, g * Sg:(g + 1) * Sg])
                else:
                    enets[g].enqueue(hnp[k, g * Sg:(g + 1) * Sg])

            def out(g, k):
                if delta:
                    enets[g].copy_output_delta(dbufs[g][k % (LAG + 1)].ptr)
                    dma.append(enets[g].last_delta_dma_bytes())
                else:
                    enets[g].copy_output_detached(out_host[g].data_ptr())

            def apply(k):  # host mirrors take step k's deltas
                list(appl.map(lambda g: enets[g].apply_output_delta(dbufs[g][k % (LAG + 1)].ptr, mirrors[g].ctypes.data),
                              range(G)))
                n = sum(int(enets[g].delta_counts(dbufs[g][k % (LAG + 1)].array).sum()) for g in range(G))
                px_bytes = out_bytes // (Sg * nodes[-1].out_shape[1] * nodes[-1].out_shape[2])  # Cs floats
                dbytes.append(G * ((4 * Sg + 15) // 16 * 16) + n * (4 + px_bytes))
            for g in range(G):
                put(g, 0)
                out(g, 0)
            for k in range(a.warmup):
                for g in range(G):
                    put(g, frame_at(k))
                    out(g, k + 1)  # staging / host buffers allocated here
            for c in ctxs:
                c.synchronize()
            if delta:
                for k in range(a.warmup + 1):
                    apply(k)
                dbytes.clear()
                dma.clear()
            barrier()

            # diagnosis only: BENCH_E2E_PROBE=noapply skips the host mirror
            # update, =noout also the delta copy (the line is then not an e2e number)
            probe = os.environ.get("BENCH_E2E_PROBE", "")
            host_t = [0.0, 0.0, 0.0]

            # the host mirrors are updated by a background thread (step k - LAG
            # while the main thread enqueues step k); a host buffer is reused
            # only after the update that read it has finished
            applier = ThreadPoolExecutor(max_workers=1) if delta else None
            pending = {}

            def e2e_step(k):
                t_a = time.perf_counter()
                if delta and (k - LAG - 1) in pending:
                    pending.pop(k - LAG - 1).result()
                for g in range(G):
                    put(g, frame_at(base_k + k))
                    if probe != "noout":
                        out(g, k)
                t_b = time.perf_counter()
                if delta and k >= LAG and not probe:
                    pending[k - LAG] = applier.submit(apply, k - LAG)
                t_c = time.perf_counter()
                host_t[0] += t_b - t_a
                host_t[1] += t_c - t_b
                host_t[2] += 1

            def finish():
                for k in sorted(pending):
                    pending.pop(k).result()
                for k in range(max(0, a.steps - LAG), a.steps):
                    apply(k)
            ems = max_over_ranks(timed_region(e2e_step, a.steps, finish if delta else None))
            if True:  # host-side cost of the loop, to stderr
                print(f"e2e probe {probe or '-'} u8={u8} delta={delta}: {ems / a.steps:.3f} ms/step device, host enqueue "
                      f"{1e3 * host_t[0] / host_t[2]:.3f} ms/step, apply {1e3 * host_t[1] / host_t[2]:.3f} ms/step",
                      file=sys.stderr)
            del enets
            r = {"value": total_streams * a.steps / (ems / 1000.0), "unit": "frames/s",
                 "h2d_bytes_per_step": frame8_bytes if u8 else frame_bytes,
                 "d2h_bytes_per_step": (sum(dma) / a.steps) if delta else out_bytes * G,
                 "ms_per_step": ems / a.steps}
            if delta:
                appl.shutdown()
                applier.shutdown()
                r["d2h_full_output_bytes"] = out_bytes * G
                r["d2h_delta_bytes_in_use"] = sum(dbytes) / len(dbytes)
            return r
        e2e = run_e2e(True, True)
        e2e["api"] = ("cbg_net_forward_u8: pinned host 8-bit PNM payloads [S][H][W][3], load_pnm conversion "
                      "(byte/255.0f) fused into the first layer's detect; result: cbg_net_copy_output_delta (the "
                      "last node's changed pixels and their output vectors, packed on the device and copied into "
                      "pinned host memory on the copy-out stream) + cbg_net_apply_output_delta into a host mirror of the full "
                      "output (the reference's whole-Tensor3 result, network.cpp:412-413), step k applied while "
                      "steps k+1..k+3 run; d2h bytes = bytes moved (DMA of the recent delta size + 25%, overflow "
                      "kernel for the rest)")
        e2e_full = run_e2e(True, False)
        e2e_full["api"] = ("as e2e, but the whole last-node output D2H every step (cbg_net_copy_output_detached: "
                           "staged on the device, copied out on the context's copy-out stream)")
        if hnp is not None:
            e2e_f32 = run_e2e(False, True)
            e2e_f32["api"] = ("cbg_net_forward: pinned host fp32 CHW frames (Tensor3); result as e2e (delta + "
                              "host mirror)")

    # ---- CPU baseline (rank 0, N=1) ---------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r = run_ref_bench(a, threads, frames=3, budget=a.cpu_budget)
        if r:
            cpu = {"value": r["fps"], "unit": "frames/s", "cores": threads, "kind": "reference",
                   "sample": f"oracle/_ref/ref_bench: {r['frames']} post-bootstrap frames of {r['streams']} "
                             f"streams, one cbi::CBNetwork per thread, L1 change "
                             f"{100 * r['l1_change_frac']:.2f}%"}
            if a.cpu_one_core_budget > 0:
                r1 = run_ref_bench(a, 1, frames=3, budget=a.cpu_one_core_budget, streams=1)
                cpu["one_core"] = {"value": r1["fps"], "unit": "frames/s", "cores": 1,
                                   "sample": f"{r1['frames']} post-bootstrap frames of 1 stream, 1 thread"}
            dpath = os.path.join(ROOT, "profiles", f"r02_cpu_dense_{a.config}.json")
            if os.path.exists(dpath):
                with open(dpath) as fh:
                    cpu["dense_oracle"] = json.load(fh)

    parity = None
    ppath = os.path.join(ROOT, "profiles", "r02_parity.json")
    if os.path.exists(ppath):
        with open(ppath) as fh:
            pj = json.load(fh).get(a.config)
        if pj:
            sm = pj["summary"]
            parity = {"source": "profiles/r02_parity.json (tests/test_gpu_fullsize.py vs oracle/_ref, "
                                "tools/parity_report.py)", "workload": pj.get("workload"),
                      "l1_bit_exact": sm.get("l1_bit_exact"), "min_mask_agreement": sm.get("min_agree"),
                      "max_rel_err": sm.get("max_rel_err"), "final_max_rel_err": sm.get("final_max_rel_err")}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": a.scaling,
               "vs_baseline": None, "dtype": "f32",
               "gemm_precision": ("3xFP16 tcgen05 kind::f16, fp32 operands split hi+lo with power-of-two scaling, "
                                  "fp32 accumulate (fp32-accurate); Cout<=16 layers bit-exact on CUDA cores"
                                  if os.environ.get("CBG_GEMM_PREC", "f16") != "tf32" else
                                  "3xTF32 tcgen05 (fp32-accurate); Cout<=16 layers bit-exact on CUDA cores"),
               "data": "synthetic (gen_synthetic, seeded; random-init He-uniform weights)",
               "config": config_dict(a, world),
               "change": {"l1_changed_frac": l1_frac, "input_detected_frac": l1_det_frac,
                          "x_axis_note": "l1_changed = the first layer's dilated output update set (its index "
                                         "list); input_detected = pixels of the frame whose |x - s| > tau "
                                         "before dilation (the paper's changed pixels, PAPER.md:213-214)",
                          "per_layer_changed_frac": per_layer},
               "dense_path_fps": dense_fps, "speedup_vs_dense": (value / dense_fps) if dense_fps else None,
               "sweep": sweep, "crossover_l1_changed_pct": crossover,
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_full_output": e2e_full, "e2e_f32": e2e_f32,
               "parity": parity,
               "gpu_launches": launches * a.steps,
               "clocks": clocks.summary()}
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
