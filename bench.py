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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=64, help="camera streams per GPU")
    ap.add_argument("--groups", type=int, default=4,
                    help="stream groups per GPU, each its own stream set on its own CUDA stream (overlap)")
    ap.add_argument("--ring", type=int, default=16, help="distinct frames per stream (ping-pong playback)")
    ap.add_argument("--height", type=int, default=480)
    ap.add_argument("--width", type=int, default=640)
    ap.add_argument("--objects", type=int, default=6)
    ap.add_argument("--object-size", type=int, default=40)
    ap.add_argument("--velocity", type=int, default=4)
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
    ap.add_argument("--sweep-steps", type=int, default=6,
                    help="timed steps per point of the change-rate sweep (0 disables the sweep)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config_dict(a, world):
    return {"workload": f"scene-labeling net (seg7 layers, derived dims) {a.width}x{a.height}, "
                        f"{a.streams} streams/GPU, gen_synthetic {a.objects}x{a.object_size}px objects "
                        f"v={a.velocity} noise={a.noise}, tau={a.tau}",
            "height": a.height, "width": a.width, "streams_per_gpu": a.streams,
            "total_streams": a.streams * world, "stream_groups": a.groups, "frame_ring": a.ring,
            "objects": a.objects, "object_size": a.object_size,
            "velocity": a.velocity, "noise_std": a.noise, "tau": a.tau,
            "frames": "gen_synthetic quantized to 8-bit PNM payloads; fp32 arms see load_pnm's byte/255.0f",
            "ingest": (f"value/roofline/dense/sweep: device-resident {getattr(a, 'ingest', 'u8')} frames "
                       "(u8 = the PNM payload through cbg_net_forward_u8, f32 = its byte/255.0f through "
                       "cbg_net_forward)"),
            "parallelism": f"streams sharded over {world} GPU(s), no collective",
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
            "warmup": a.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
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
# algorithmic work per kernel
# ---------------------------------------------------------------------------
def kernel_work(node, kernel, n_out, n_up, S_counts):
    """Algorithmic (bytes, flops) of one launch, summed over the streams.
    n_out/n_up: per-stream lists of this node's / its producer's changed pixels."""
    kind, name, cin, hin, win, cout, hout, wout, k, ops_pp = node
    b = f = 0.0
    for s in range(S_counts):
        no = int(n_out[s])
        nu = int(n_up[s]) if n_up is not None else None
        if kernel == "detect":
            if nu is None:  # dense scan of the network input: read x and state
                b += 8.0 * cin * hin * win
            else:           # sparse: x and state at the producer's update set
                b += 8.0 * cin * nu
        elif kernel == "dilcomp":
            b += hin * win / 8.0 + hout * wout / 8.0 + 4.0 * no + 4
        elif kernel == "gemm":
            f += ops_pp * no
            # gather lower bound (each changed pixel's own receptive-field centre),
            # weights once, scatter of the Cout vector
            b += 4.0 * cin * no + 4.0 * cout * no + (4.0 * cout * cin * k * k if s == 0 else 0.0)
        elif kernel == "pool":
            b += 4.0 * cin * 4 * no + 4.0 * cin * no
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
    from paper_1808_05488_b200.sharding import weak_shard

    peaks = {"hbm_gbs": 6538.6, "bf16_tflops": 1661.9, "bf16_tflops_sustained": 1399.9, "source": "fallback"}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        with open(pk_path) as fh:
            peaks.update(json.load(fh))
        peaks["source"] = "measured (MEASURED_PEAKS.json)"

    S, H, W, G = a.streams, a.height, a.width, a.groups
    if S % G:
        raise SystemExit("--streams must be a multiple of --groups")
    Sg = S // G
    ctxs = [cbi.Context(local) for _ in range(G)]
    ctx = ctxs[0]
    spec = cbi.make_seg_spec(1, H, W)
    taus = [a.tau] * 5
    L = max(3, a.ring)
    # frame ring [L][S][C][H][W], pinned on the host and resident in HBM; played
    # ping-pong (1..L-1, L-2..2, ...) so motion stays continuous for any step count
    # The frames are what a PNM sequence delivers (cbi run -> load_pnm): 8-bit
    # payloads ([H][W][C] bytes) of gen_synthetic frames; the fp32 arm sees
    # load_pnm's byte / 255.0f of the same bytes, so every arm runs one workload.
    host = torch.empty((L, S, 3, H, W), dtype=torch.float32, pin_memory=True)
    host8 = torch.empty((L, S, H, W, 3), dtype=torch.uint8, pin_memory=True)
    hnp, h8np = host.numpy(), host8.numpy()
    shard = weak_shard(S, rank, world)  # streams rank*S .. rank*S+S-1, seed 1000 + global id
    for s in range(S):
        raw = cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, L, a.objects, a.object_size, a.velocity,
                                                    a.velocity, a.noise, shard.seed(s)))
        h8np[:, s] = cbi.to_pnm8(raw)
        hnp[:, s] = cbi.from_pnm8(h8np[:, s])
    dev = host.to(f"cuda:{local}")
    dev8 = host8.to(f"cuda:{local}")
    torch.cuda.synchronize()
    u8_in = a.ingest == "u8"

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
    nodes = net.nodes()
    counts_pinned = torch.empty((G, a.steps + 1, n_slots, Sg), dtype=torch.int32, pin_memory=True)

    def dptr(t, g):
        return dev[t, g * Sg].data_ptr()

    def timed_region(step_fn, steps):
        """device time of `steps` calls of step_fn(k) across all groups (CUDA events)"""
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(ext)
        for e in exts[1:]:
            e.wait_event(t0)
        for k in range(steps):
            step_fn(k)
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
    cnt = np.concatenate([counts_pinned[g, :a.steps].numpy() for g in range(G)], axis=2)
    l1_px = nodes[0].out_shape[1] * nodes[0].out_shape[2]
    l1_frac = float(cnt[:, node_slot[0], :].mean()) / l1_px
    per_layer = {n.name: float(cnt[:, node_slot[i], :].mean()) / (n.out_shape[1] * n.out_shape[2])
                 for i, n in enumerate(nodes)}
    value = S * world * a.steps / (ms / 1000.0)
    next_k = base_k + a.steps

    # ---- roofline: instrumented pass (per-kernel CUDA events) -----------------
    # one stream set holding all S streams (the launch shape of the ncu capture
    # in profiles/), eager launches with an event pair around every kernel
    pnet = cbi.convert_to_cb(spec, taus, n_streams=S, ctx=ctx)
    feed(pnet, 0)
    for k in range(2):
        feed(pnet, frame_at(next_k + k))
    ctx.synchronize()
    pnet.set_kernel_timing(True)
    work = {}
    prof_counts = torch.empty((n_slots, S), dtype=torch.int32, pin_memory=True)
    for k in range(a.profile_steps):
        feed(pnet, frame_at(next_k + 2 + k))
        pnet.copy_counts_async(prof_counts.data_ptr())
        ctx.synchronize()
        c = prof_counts.numpy()
        for i, n in enumerate(nodes):
            src = n.inputs[0] if n.inputs else -1
            cin, hin, win = n.in_shape
            cout, hout, wout = n.out_shape
            kk = 0
            if n.kind == cbi.LayerKind.Conv:
                kk = int(round((n.ops_per_pixel / (2 * cout * max(1, cin))) ** 0.5))
            desc = (n.kind, n.name, cin, hin, win, cout, hout, wout, kk, int(n.ops_per_pixel))
            n_out = c[node_slot[i]]
            n_up = c[node_slot[src]] if src >= 0 else None
            for kern in ("detect", "dilcomp", "gemm", "pool"):
                bb, ff = kernel_work(desc, kern, n_out, n_up, S)
                wsum = work.setdefault(f"{n.name}.{kern}", [0.0, 0.0])
                wsum[0] += bb
                wsum[1] += ff
    rep = pnet.timing_report()
    pnet.set_kernel_timing(False)
    del pnet
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if tj.get("streams") == S and tj.get("height") == H and tj.get("width") == W:
            traffic = tj.get("dram_bytes_per_launch", {})
    hbm = peaks["hbm_gbs"] * 1e9
    # the tcgen05 GEMMs run kind::f16 (3xFP16 split, default) or kind::tf32
    # (CBG_GEMM_PREC=tf32); the tensor peak is that kind's dense rate: the
    # measured bf16 (= fp16) rate, or half of it for tf32
    f16_gemm = os.environ.get("CBG_GEMM_PREC", "f16") != "tf32"
    tf32 = peaks["bf16_tflops"] * 1e12 / (1 if f16_gemm else 2)
    kernels = []
    for label, (tot_ms, nl) in rep["kernels"].items():
        bb, ff = work.get(label, [0.0, 0.0])
        t = tot_ms / 1000.0
        t_roof = max(bb / hbm, ff / tf32)
        kernels.append({"kernel": label, "ms_per_launch": tot_ms / max(1, nl), "share": 0.0,
                        "bytes_per_launch": bb / max(1, nl), "flops_per_launch": ff / max(1, nl),
                        "roofline_frac": (t_roof / t) if t > 0 else None,
                        "bound": "tensor" if ff / tf32 > bb / hbm else "hbm"})
    tot = sum(k["ms_per_launch"] for k in kernels) or 1.0
    for k in kernels:
        k["share"] = k["ms_per_launch"] / tot
    kernels.sort(key=lambda k: -k["ms_per_launch"])
    dom = kernels[0]
    if dom["bound"] == "tensor":
        achieved = dom["flops_per_launch"] / (dom["ms_per_launch"] / 1000.0) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tf32 / 1e12, "unit": "TFLOP/s",
                "frac": achieved / (tf32 / 1e12),
                # the split-fp32 product issues 3 MMAs per useful MAC: the tensor
                # pipe's share is 3x the useful fraction (attainable useful frac <= 1/3)
                "tensor_issue_frac": 3 * achieved / (tf32 / 1e12),
                "peak_note": ("fp16 dense = measured bf16 rate" if f16_gemm else "tf32 dense = measured bf16 / 2")
                + "; useful fp32-accurate flops (2*Cout*Cin*k^2 per changed px), 3 MMAs per useful MAC"}
    else:
        achieved = dom["bytes_per_launch"] / (dom["ms_per_launch"] / 1000.0) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    roof.update({"kernel": dom["kernel"], "traffic": traffic.get(dom["kernel"]),
                 "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, profiles/ncu_traffic.json",
                 "launch_streams": S, "peak_source": peaks["source"],
                 "step_roofline_frac": (sum(max(k["bytes_per_launch"] / hbm, k["flops_per_launch"] / tf32)
                                            for k in kernels) / (tot / 1000.0)),
                 "top_kernels": kernels[:6],
                 "all_kernels_us": {k["kernel"]: round(1000 * k["ms_per_launch"], 1) for k in kernels}})

    # ---- dense path (same kernels, every frame a full update) -------------------
    dense_fps = None
    if a.dense_steps > 0:
        dnets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
        for g in range(G):
            dnets[g].set_dense(True)
            feed(dnets[g], 0, g)
            feed(dnets[g], 1, g)
        for c in ctxs:
            c.synchronize()

        def dense_step(k):
            for g in range(G):
                feed(dnets[g], frame_at(k), g)

        dms = max_over_ranks(timed_region(dense_step, a.dense_steps))
        dense_fps = S * world * a.dense_steps / (dms / 1000.0)
        del dnets

    # ---- change-rate sweep: frames/s vs changed-pixel % (the metric's x-axis) ---
    sweep = []
    if a.sweep_steps > 0:
        from concurrent.futures import ThreadPoolExecutor
        R = 6
        sorder = list(range(1, R)) + list(range(R - 2, 1, -1))
        sw_counts = torch.empty((G, n_slots, Sg), dtype=torch.int32, pin_memory=True)
        for pt in SWEEP:
            if pt == "random":
                gen = torch.Generator(device=f"cuda:{local}").manual_seed(4242 + rank)
                if u8_in:
                    sdev = torch.randint(0, 256, (R, S, H, W, 3), generator=gen, device=f"cuda:{local}",
                                         dtype=torch.uint8)
                else:
                    sdev = torch.rand((R, S, 3, H, W), generator=gen, device=f"cuda:{local}")
            else:
                ob, sz = pt
                sh = torch.empty((R, S, H, W, 3) if u8_in else (R, S, 3, H, W),
                                 dtype=torch.uint8 if u8_in else torch.float32, pin_memory=True)
                shn = sh.numpy()

                def _gen(s_, ob=ob, sz=sz, shn=shn):
                    p8 = cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(
                        H, W, 3, R, ob, sz, a.velocity, a.velocity, a.noise, shard.seed(s_))))
                    shn[:, s_] = p8 if u8_in else cbi.from_pnm8(p8)
                with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
                    list(pool.map(_gen, range(S)))
                sdev = sh.to(f"cuda:{local}")

            def sfeed(net_, t, g, sdev=None):
                if u8_in:
                    net_.enqueue_device_u8(sdev[t, g * Sg].data_ptr())
                else:
                    net_.enqueue_device(sdev[t, g * Sg].data_ptr())
            snets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
            for g in range(G):
                sfeed(snets[g], 0, g, sdev)
            for k in range(3):
                for g in range(G):
                    sfeed(snets[g], sorder[k % len(sorder)], g, sdev)
            for c in ctxs:
                c.synchronize()
            barrier()

            def sweep_step(k, snets=snets, sdev=sdev):
                for g in range(G):
                    sfeed(snets[g], sorder[(3 + k) % len(sorder)], g, sdev)

            sms = max_over_ranks(timed_region(sweep_step, a.sweep_steps))
            for g in range(G):
                snets[g].copy_counts_async(sw_counts[g].data_ptr())
            for c in ctxs:
                c.synchronize()
            sc = np.concatenate([sw_counts[g].numpy() for g in range(G)], axis=1)
            fps = S * world * a.sweep_steps / (sms / 1000.0)
            sweep.append({"synthetic": ("uniform noise every frame" if pt == "random"
                                        else f"{pt[0]} objects x {pt[1]} px"),
                          "l1_changed_pct": 100.0 * float(sc[node_slot[0]].mean()) / l1_px,
                          "per_layer_changed_pct": {n.name: round(100.0 * float(sc[node_slot[i]].mean())
                                                                  / (n.out_shape[1] * n.out_shape[2]), 3)
                                                    for i, n in enumerate(nodes)},
                          "frames_per_s": fps,
                          "speedup_vs_dense": (fps / dense_fps) if dense_fps else None})
            del snets, sdev
        torch.cuda.empty_cache()
    crossover = None
    if dense_fps and sweep:
        pts = sorted((p["l1_changed_pct"], p["frames_per_s"] / dense_fps) for p in sweep)
        for (x0, r0), (x1, r1) in zip(pts, pts[1:]):
            if r0 >= 1.0 > r1:  # linear in log(change) between the bracketing points
                import math
                f = (r0 - 1.0) / (r0 - r1)
                crossover = math.exp(math.log(max(x0, 1e-6)) + f * (math.log(x1) - math.log(max(x0, 1e-6))))
                break

    # ---- e2e: host frames through the C ABI, H2D + D2H in the timed region -------
    # headline: 8-bit PNM payloads (cbg_net_forward_u8, load_pnm's conversion on
    # the device); also the fp32 Tensor3 API (cbg_net_forward) with host frames
    e2e = e2e_f32 = None
    if not a.no_e2e:
        def run_e2e(u8):
            enets = [cbi.convert_to_cb(spec, taus, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
            out_bytes = enets[0].output_bytes(-1)
            out_host = [torch.empty(out_bytes // 4, dtype=torch.float32, pin_memory=True) for _ in range(G)]

            def put(g, k):
                if u8:
                    enets[g].enqueue_u8(h8np[k, g * Sg:(g + 1) * Sg])
                else:
                    enets[g].enqueue(hnp[k, g * Sg:(g + 1) * Sg])
            for g in range(G):
                put(g, 0)
            for k in range(a.warmup):
                for g in range(G):
                    put(g, frame_at(k))
                    enets[g].copy_output_detached(out_host[g].data_ptr())  # staging buffers allocated here
            for c in ctxs:
                c.synchronize()
            barrier()

            def e2e_step(k):
                for g in range(G):
                    put(g, frame_at(base_k + k))
                    enets[g].copy_output_detached(out_host[g].data_ptr())

            ems = max_over_ranks(timed_region(e2e_step, a.steps))
            del enets
            return {"value": S * world * a.steps / (ems / 1000.0), "unit": "frames/s",
                    "h2d_bytes_per_step": frame8_bytes if u8 else frame_bytes, "d2h_bytes_per_step": out_bytes * G,
                    "ms_per_step": ems / a.steps}
        e2e = run_e2e(True)
        e2e["api"] = ("cbg_net_forward_u8: pinned host 8-bit PNM payloads [S][H][W][3], load_pnm conversion "
                      "(byte/255.0f) fused into the first layer's detect; D2H of the last node's output (cbg_net_copy_output_detached: "
                      "staged on the device, copied out on the context's copy-out stream)")
        e2e_f32 = run_e2e(False)
        e2e_f32["api"] = ("cbg_net_forward: pinned host fp32 CHW frames (Tensor3); D2H of the last node's output "
                          "(cbg_net_copy_output_detached)")

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

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32",
               "gemm_precision": ("3xFP16 tcgen05 kind::f16, fp32 operands split hi+lo with power-of-two scaling, "
                                  "fp32 accumulate (fp32-accurate); Cout<=16 layers bit-exact on CUDA cores"
                                  if os.environ.get("CBG_GEMM_PREC", "f16") != "tf32" else
                                  "3xTF32 tcgen05 (fp32-accurate); Cout<=16 layers bit-exact on CUDA cores"),
               "data": "synthetic (gen_synthetic, seeded; random-init He-uniform weights)",
               "config": config_dict(a, world),
               "change": {"l1_changed_frac": l1_frac, "per_layer_changed_frac": per_layer},
               "dense_path_fps": dense_fps, "speedup_vs_dense": (value / dense_fps) if dense_fps else None,
               "sweep": sweep, "crossover_l1_changed_pct": crossover,
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_f32": e2e_f32,
               "gpu_launches": launches * a.steps,
               "clocks": clocks.summary()}
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
