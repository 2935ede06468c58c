"""Python mirror of the reference ``cbi`` layer API, backed by the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/cbi/{tensor,change,layers,network,io}.hpp), so
parity tests read like the reference's own tests. Every compute call goes
through ``libcbg.so`` (hand-written sm_100a kernels); nothing here computes on
the CPU except the host-side harness generators the reference also ships
(gen_synthetic / fill_random_weights, mirrored in C++ inside libcbg).

Data conventions (reference tensor.hpp / change.hpp):
  Tensor3    -> numpy float32 array [C, H, W]
  ChangeMap  -> numpy uint8 array [H, W] (0/1)
  IndexList  -> numpy int32 array [n, 2] of (row, col), row-major order
"""
from __future__ import annotations

import ctypes as C
import json
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (ConfigError, InvalidInputError, check, fptr, lib)

__all__ = [
    "LayerKind", "DetectionPolicy", "DetectMode", "ConvSpec", "LayerDesc", "NetworkSpec",
    "SyntheticConfig", "UpstreamChange", "ConvForwardResult", "PoolForwardResult", "StatsConfig",
    "LayerFrameStats", "FrameStats", "RunStats", "SequenceResult", "Context", "CBConvLayer",
    "CBPoolLayer", "CBNetwork", "convert_to_cb", "validate_network", "forward_sequence", "write_stats_csv",
    "loss_value", "select_thresholds", "sweep_threshold_factor",
    "gen_synthetic", "fill_random_weights", "make_seg7_spec", "make_seg_spec", "make_small_spec", "make_yolov3_spec",
    "InvalidInputError", "ConfigError", "device_available",
]


class LayerKind(enum.IntEnum):  # network.hpp:10
    Conv = _lib.LAYER_CONV
    Act = _lib.LAYER_ACT
    Pool = _lib.LAYER_POOL
    Add = _lib.LAYER_ADD
    Concat = _lib.LAYER_CONCAT
    Upsample = _lib.LAYER_UPSAMPLE  # extension: not in the reference


class DetectionPolicy(enum.IntEnum):  # layers.hpp:8
    Detect = _lib.POLICY_DETECT
    Propagate = _lib.POLICY_PROPAGATE
    Reuse1x1 = _lib.POLICY_REUSE1X1


class DetectMode(enum.IntEnum):  # change.hpp:34
    FeedForward = _lib.MODE_FEEDFORWARD
    ClosedLoop = _lib.MODE_CLOSEDLOOP


def device_available() -> bool:
    return bool(lib.cbg_device_available())


# ---------------------------------------------------------------------------
# descriptions
# ---------------------------------------------------------------------------
@dataclass
class ConvSpec:
    """ConvSpec, tensor.hpp:54-80. weights [out][in][kh][kw], bias [out]."""

    in_channels: int = 0
    out_channels: int = 0
    kernel_h: int = 0
    kernel_w: int = 0
    stride: int = 1
    padding: int = 0
    out_h: int = 0
    out_w: int = 0
    weights: Optional[np.ndarray] = None
    bias: Optional[np.ndarray] = None

    def weight_count(self) -> int:
        return self.out_channels * self.in_channels * self.kernel_h * self.kernel_w

    def output_height(self, in_h: int) -> int:  # tensor.cpp:22-24
        return self.out_h if self.out_h > 0 else _derived(in_h, self.kernel_h, self.stride, self.padding)

    def output_width(self, in_w: int) -> int:  # tensor.cpp:26-28
        return self.out_w if self.out_w > 0 else _derived(in_w, self.kernel_w, self.stride, self.padding)

    def _c(self, keep: list) -> _lib.ConvSpecC:
        w = np.ascontiguousarray(self.weights if self.weights is not None else
                                 np.zeros(max(self.weight_count(), 0), np.float32), dtype=np.float32)
        b = np.ascontiguousarray(self.bias if self.bias is not None else
                                 np.zeros(max(self.out_channels, 0), np.float32), dtype=np.float32)
        if w.size != self.weight_count():
            raise InvalidInputError(f"conv spec: weight count {w.size} != out*in*kh*kw = {self.weight_count()}")
        if b.size != self.out_channels:
            raise InvalidInputError(f"conv spec: bias count {b.size} != out_channels = {self.out_channels}")
        keep += [w, b]
        return _lib.ConvSpecC(self.in_channels, self.out_channels, self.kernel_h, self.kernel_w,
                              self.stride, self.padding, self.out_h, self.out_w,
                              w.ctypes.data_as(C.POINTER(C.c_float)), b.ctypes.data_as(C.POINTER(C.c_float)))


def _derived(in_dim, k, s, p):  # tensor.cpp:9-20
    v = (in_dim + 2 * p - k) // s + 1
    if in_dim + 2 * p - k < 0 or v < 1:
        raise InvalidInputError(f"conv output dim < 1 (input {in_dim}, kernel {k}, stride {s}, padding {p})")
    return v


@dataclass
class LayerDesc:
    """LayerDesc, network.hpp:25-37."""

    kind: LayerKind = LayerKind.Conv
    name: str = ""
    from_: List[str] = field(default_factory=list)
    conv: ConvSpec = field(default_factory=ConvSpec)
    fuse_relu: bool = False
    pool_size: int = 0
    pool_stride: int = 0
    pool_out_h: int = 0
    pool_out_w: int = 0
    act_slope: float = 0.0  # extension: leaky ReLU slope of an Act row / a conv's fused act (0 = ReLU)
    upsample: int = 0       # extension: Upsample rows' factor


@dataclass
class NetworkSpec:
    """NetworkSpec, network.hpp:39-44."""

    in_channels: int = 0
    in_height: int = 0
    in_width: int = 0
    layers: List[LayerDesc] = field(default_factory=list)

    def _c(self, keep: list) -> _lib.NetworkSpecC:
        arr = (_lib.LayerDescC * max(1, len(self.layers)))()
        for i, d in enumerate(self.layers):
            names = [s.encode() for s in d.from_]
            from_arr = (C.c_char_p * max(1, len(names)))(*names)
            name = d.name.encode()
            keep += [names, from_arr, name]
            conv = d.conv._c(keep) if d.kind == LayerKind.Conv else _lib.ConvSpecC()
            arr[i] = _lib.LayerDescC(int(d.kind), name, len(names), from_arr, conv, int(bool(d.fuse_relu)),
                                     d.pool_size, d.pool_stride, d.pool_out_h, d.pool_out_w,
                                     float(d.act_slope), int(d.upsample))
        keep.append(arr)
        return _lib.NetworkSpecC(self.in_channels, self.in_height, self.in_width, len(self.layers), arr)


@dataclass
class SyntheticConfig:
    """SyntheticConfig, io.hpp:47-58."""

    height: int = 128
    width: int = 128
    channels: int = 3
    n_frames: int = 20
    n_objects: int = 2
    object_size: int = 8
    velocity_y: int = 1
    velocity_x: int = 1
    noise_std: float = 0.0
    seed: int = 1


def gen_synthetic(cfg: SyntheticConfig, with_corners: bool = False):
    """gen_synthetic, io.cpp:499-552 -> array [n_frames, C, H, W] (and corners)."""
    c = _lib.SyntheticConfigC(cfg.height, cfg.width, cfg.channels, cfg.n_frames, cfg.n_objects,
                              cfg.object_size, cfg.velocity_y, cfg.velocity_x, cfg.noise_std, cfg.seed)
    frames = np.empty((max(cfg.n_frames, 0), max(cfg.channels, 0), max(cfg.height, 0), max(cfg.width, 0)),
                      np.float32)
    corners = np.empty((max(cfg.n_frames, 0), max(cfg.n_objects, 0), 2), np.int32) if with_corners else None
    check(lib.cbg_gen_synthetic(C.byref(c), fptr(frames), fptr(corners)))
    return (frames, corners) if with_corners else frames


# ---------------------------------------------------------------------------
# threshold calibration on the GPU (calibration.hpp:16-84)
# ---------------------------------------------------------------------------
class LossMetric(enum.IntEnum):  # network.hpp:183
    Mse = 0
    PixelAccuracyDelta = 1


class LossAggregation(enum.IntEnum):  # calibration.hpp:26
    Mean = 0
    Worst = 1


@dataclass
class EvalSequence:
    """EvalSequence, calibration.hpp:19-22: frames [n, C, H, W] and one reference
    output per frame ([n, Co, Ho, Wo], or [n, 1, Ho, Wo] class labels)."""

    frames: np.ndarray
    reference: np.ndarray


@dataclass
class CalibConfig:  # calibration.hpp:28-36
    initial_tau: float = 0.01
    growth_factor: float = 1.1
    per_layer_budget: float = 0.0
    budget_overrides: List[float] = field(default_factory=list)
    metric: LossMetric = LossMetric.Mse
    aggregation: LossAggregation = LossAggregation.Mean
    max_steps: int = 64


@dataclass
class CalibTracePoint:  # calibration.hpp:38-42
    layer: int
    tau: float
    loss: float


@dataclass
class CalibResult:  # calibration.hpp:44-48
    taus: List[float]
    hit_cap: List[bool]
    trace: List[CalibTracePoint]


@dataclass
class TradeoffRow:  # calibration.hpp:56-61
    factor: float
    loss: float
    total_eff_ops: int
    wall_ns: int


def _sequences_c(sequences, keep):
    arr = (_lib.EvalSequenceC * max(1, len(sequences)))()
    for i, q in enumerate(sequences):
        f = np.ascontiguousarray(q.frames, dtype=np.float32)
        r = np.ascontiguousarray(q.reference, dtype=np.float32)
        if r.ndim != 4 or f.ndim != 4 or len(r) != len(f):
            raise InvalidInputError("calibration sequence needs frames and per-frame references")
        keep += [f, r]
        arr[i] = _lib.EvalSequenceC(len(f), f.ctypes.data, r.ctypes.data, r.shape[1])
    keep.append(arr)
    return arr


def select_thresholds(net: "CBNetwork", sequences: Sequence[EvalSequence], cfg: CalibConfig = None) -> CalibResult:
    """select_thresholds (calibration.cpp:95-141) with every candidate's replay on
    the GPU (one stream per candidate, cbg_select_thresholds). ``net`` supplies the
    topology, policies and mode."""
    cfg = cfg or CalibConfig()
    keep: list = []
    seqs = _sequences_c(list(sequences), keep)
    ov = np.ascontiguousarray(cfg.budget_overrides, dtype=np.float64)
    c = _lib.CalibConfigC(cfg.initial_tau, cfg.growth_factor, cfg.per_layer_budget,
                          ov.ctypes.data if len(ov) else None, len(ov), int(cfg.metric), int(cfg.aggregation),
                          cfg.max_steps)
    n_conv = net.conv_layer_count()
    taus = np.zeros(n_conv, np.float32)
    cap = np.zeros(n_conv, np.uint8)
    cap_trace = max(1, n_conv * max(1, cfg.max_steps))
    trace = (_lib.CalibTracePointC * cap_trace)()
    n = C.c_int(0)
    check(lib.cbg_select_thresholds(net.handle, seqs, len(sequences), C.byref(c), fptr(taus),
                                    cap.ctypes.data_as(C.c_void_p), trace, cap_trace, C.byref(n)))
    return CalibResult([float(t) for t in taus], [bool(x) for x in cap],
                       [CalibTracePoint(trace[i].layer, trace[i].tau, trace[i].loss) for i in range(min(n.value,
                                                                                                       cap_trace))])


def sweep_threshold_factor(net: "CBNetwork", base_tau: Sequence[float], factors: Sequence[float],
                           sequences: Sequence[EvalSequence], metric: LossMetric = LossMetric.Mse) -> List[TradeoffRow]:
    """sweep_threshold_factor (calibration.cpp:143-180), one stream per factor on the GPU."""
    keep: list = []
    seqs = _sequences_c(list(sequences), keep)
    bt = np.ascontiguousarray(base_tau, dtype=np.float32)
    fa = np.ascontiguousarray(factors, dtype=np.float64)
    rows = (_lib.TradeoffRowC * max(1, len(fa)))()
    check(lib.cbg_sweep_threshold_factor(net.handle, fptr(bt), len(bt), fa.ctypes.data_as(C.c_void_p), len(fa), seqs,
                                         len(sequences), int(metric), rows))
    return [TradeoffRow(rows[i].factor, rows[i].loss, rows[i].total_eff_ops, rows[i].wall_ns) for i in range(len(fa))]


def to_pnm8(frames: np.ndarray) -> np.ndarray:
    """8-bit PNM payload ([..., H, W, C] uint8) of planar fp32 frames ([..., C, H, W]):
    byte = floor(clamp(v, 0, 1) * 255 + 0.5) in fp32 (what a camera / PNM writer
    would store; the reference has no writer, only load_pnm)."""
    f = np.clip(np.asarray(frames, np.float32), np.float32(0), np.float32(1))
    q = np.floor(f * np.float32(255.0) + np.float32(0.5)).astype(np.uint8)
    return np.ascontiguousarray(np.moveaxis(q, -3, -1))


def from_pnm8(payload: np.ndarray) -> np.ndarray:
    """load_pnm's conversion (io.cpp:389-397): [..., H, W, C] bytes -> [..., C, H, W] fp32 = byte / 255.0f."""
    return np.ascontiguousarray(np.moveaxis(np.asarray(payload, np.uint8).astype(np.float32) / np.float32(255.0),
                                            -1, -3))


def fill_random_weights(spec: NetworkSpec, seed: int) -> None:
    """fill_random_weights, io.cpp:554-566 (in place)."""
    convs = [d for d in spec.layers if d.kind == LayerKind.Conv]
    for d in convs:
        d.conv.weights = np.zeros(d.conv.weight_count(), np.float32)
        d.conv.bias = np.zeros(d.conv.out_channels, np.float32)
    keep: list = []
    cspec = spec._c(keep)
    W = (C.c_void_p * max(1, len(convs)))(*[d.conv.weights.ctypes.data for d in convs])
    B = (C.c_void_p * max(1, len(convs)))(*[d.conv.bias.ctypes.data for d in convs])
    check(lib.cbg_fill_random_weights(C.byref(cspec), seed, W, B))


def _conv(name, cin, cout, k, pad, relu, oh=0, ow=0, stride=1, slope=0.0, from_=None):
    return LayerDesc(LayerKind.Conv, name, list(from_ or []), ConvSpec(cin, cout, k, k, stride, pad, oh, ow), relu,
                     act_slope=slope)


def _act(name):
    return LayerDesc(LayerKind.Act, name)


def _pool(name, oh=0, ow=0):
    return LayerDesc(LayerKind.Pool, name, pool_size=2, pool_stride=2, pool_out_h=oh, pool_out_w=ow)


def make_seg7_spec(seed: int) -> NetworkSpec:
    """make_seg7_spec, io.cpp:568-617: the paper's scene-labeling net, pinned 776x1040 dims."""
    spec = NetworkSpec(3, 776, 1040, [
        _conv("L1", 3, 16, 7, 0, False, 541, 871), _act("L2a"), _pool("L2b", 271, 436),
        _conv("L3", 16, 64, 7, 3, False, 271, 436), _act("L4a"), _pool("L4b", 136, 218),
        _conv("L5", 64, 256, 7, 3, True, 136, 218), _conv("L6", 256, 64, 1, 0, True, 136, 218),
        _conv("L7", 64, 8, 1, 0, False, 136, 218)])
    fill_random_weights(spec, seed)
    return spec


def make_seg_spec(seed: int, height: int, width: int) -> NetworkSpec:
    """The same layer list with derived (unpinned) dims at any resolution."""
    spec = NetworkSpec(3, height, width, [
        _conv("L1", 3, 16, 7, 0, False), _act("L2a"), _pool("L2b"),
        _conv("L3", 16, 64, 7, 3, False), _act("L4a"), _pool("L4b"),
        _conv("L5", 64, 256, 7, 3, True), _conv("L6", 256, 64, 1, 0, True),
        _conv("L7", 64, 8, 1, 0, False)])
    fill_random_weights(spec, seed)
    return spec


def make_openpose_spec(seed: int, height: int = 368, width: int = 368, width_div: int = 1,
                       stages: int = 2) -> NetworkSpec:
    """OpenPose-style pose net (BASELINE configs[2]) as a reference layer manifest
    (conv / pool / concat with ``from=`` producers, network.hpp:25-44, io.hpp:14-22):
    the VGG-19 front end (conv1_1 .. conv4_2) + conv4_3/4_4 "CPM" layers -> features
    F, stage 1 = two branches (PAF: 38 maps, heatmaps: 19 maps) of 3x3 convs and 1x1
    heads, stage t >= 2 = concat(PAF_{t-1}, heat_{t-1}, F) -> two branches of 7x7
    convs. ReLU after every conv except the heads. Channel widths are divided by
    ``width_div`` (heads keep 38 / 19) so the CPU reference can check it quickly."""
    def ch(c):
        return max(4, c // width_div)

    L = []
    def conv(name, cin, cout, k, relu=True, frm=None):
        d = _conv(name, cin, cout, k, k // 2, relu)
        if frm:
            d.from_ = list(frm)
        L.append(d)
        return cout

    c = conv("conv1_1", 3, ch(64), 3)
    c = conv("conv1_2", c, ch(64), 3)
    L.append(_pool("pool1"))
    c = conv("conv2_1", c, ch(128), 3)
    c = conv("conv2_2", c, ch(128), 3)
    L.append(_pool("pool2"))
    c = conv("conv3_1", c, ch(256), 3)
    for i in (2, 3, 4):
        c = conv(f"conv3_{i}", c, ch(256), 3)
    L.append(_pool("pool3"))
    c = conv("conv4_1", c, ch(512), 3)
    c = conv("conv4_2", c, ch(512), 3)
    c = conv("conv4_3_CPM", c, ch(256), 3)
    feat = conv("conv4_4_CPM", c, ch(128), 3)
    prev = None
    for t in range(1, stages + 1):
        heads = []
        for br, n_out in ((1, 38), (2, 19)):
            src = ["conv4_4_CPM"] if t == 1 else [f"concat_stage{t}"]
            if t > 1 and br == 1:
                L.append(LayerDesc(LayerKind.Concat, f"concat_stage{t}", list(prev) + ["conv4_4_CPM"]))
            cin = feat if t == 1 else 38 + 19 + feat
            k, n_mid = (3, 3) if t == 1 else (7, 5)
            x = conv(f"Mconv1_stage{t}_L{br}", cin, ch(128), k, frm=src)
            for i in range(2, n_mid + 1):
                x = conv(f"Mconv{i}_stage{t}_L{br}", x, ch(128), k)
            x = conv(f"Mconv{n_mid + 1}_stage{t}_L{br}", x, ch(512) if t == 1 else ch(128), 1)
            conv(f"Mconv{n_mid + 2}_stage{t}_L{br}", x, n_out, 1, relu=False)
            heads.append(f"Mconv{n_mid + 2}_stage{t}_L{br}")
        prev = heads
    spec = NetworkSpec(3, height, width, L)
    fill_random_weights(spec, seed)
    return spec


def make_yolo_spec(seed: int, height: int = 1080, width: int = 1920, width_div: int = 1) -> NetworkSpec:
    """YOLO-style detector (BASELINE configs[3]): the tiny-YOLOv2 layer stack
    (3x3 convs 16..1024 with 2x2 / stride-2 max-pools, then a 1x1 head of 5
    anchors x (5 + 20 classes) = 125 maps). The reference has ReLU only
    (network.hpp:10), so ReLU stands in for the leaky ReLU; widths are divided by
    ``width_div`` (head kept) for the CPU-checked tests."""
    def ch(c):
        return max(4, c // width_div)

    L = []
    c = 3
    for i, cout in enumerate((16, 32, 64, 128, 256)):
        L.append(_conv(f"conv{i + 1}", c, ch(cout), 3, 1, True))
        L.append(_pool(f"pool{i + 1}"))
        c = ch(cout)
    L.append(_conv("conv6", c, ch(512), 3, 1, True))
    L.append(_conv("conv7", ch(512), ch(1024), 3, 1, True))
    L.append(_conv("conv8", ch(1024), ch(1024), 3, 1, True))
    L.append(_conv("head", ch(1024), 125, 1, 0, False))
    spec = NetworkSpec(3, height, width, L)
    fill_random_weights(spec, seed)
    return spec


def make_yolov3_spec(seed: int, height: int = 1080, width: int = 1920, width_div: int = 1,
                     slope: float = 0.1) -> NetworkSpec:
    """YOLOv3-style two-scale detector (BASELINE configs[3], the tiny-YOLOv3 layer
    graph): 3x3 convs 16..1024 with leaky ReLU (slope 0.1) and 2x2 / stride-2
    max-pools, a 1/32 head, and a route back from the 1x1 bottleneck through a
    1x1 conv and a x2 nearest upsampling, concatenated with the 1/16 features,
    to a second head; heads are linear 1x1 convs of 3 anchors x (5 + 80 classes).
    Leaky ReLU and upsampling are extensions (the reference has neither,
    network.hpp:10): they are checked against oracle/cbi_oracle.c only. Pools are
    ceil-mode (pinned output dims) and the upsampling is cropped to the 1/16
    dims, so the route meets them at any input size (1920x1080: 68x120).
    Widths are divided by ``width_div`` (heads kept)."""
    def ch(c):
        return max(4, c // width_div)

    def up2(x):
        return (x + 1) // 2

    L = []
    c, h, w = 3, height, width
    for i, cout in enumerate((16, 32, 64, 128, 256)):
        L.append(_conv(f"conv{i + 1}", c, ch(cout), 3, 1, True, slope=slope))
        if i == 4:
            h16, w16 = h, w  # conv5's dims: the route's partner
        h, w = up2(h), up2(w)
        L.append(_pool(f"pool{i + 1}", h, w))
        c = ch(cout)
    L.append(_conv("conv6", c, ch(512), 3, 1, True, slope=slope))
    L.append(_conv("conv7", ch(512), ch(1024), 3, 1, True, slope=slope))
    L.append(_conv("conv8", ch(1024), ch(256), 1, 0, True, slope=slope))
    L.append(_conv("conv9", ch(256), ch(512), 3, 1, True, slope=slope))
    L.append(_conv("head1", ch(512), 255, 1, 0, False))
    L.append(_conv("conv10", ch(256), ch(128), 1, 0, True, slope=slope, from_=["conv8"]))
    L.append(LayerDesc(LayerKind.Upsample, "up", upsample=2, pool_out_h=h16, pool_out_w=w16))
    L.append(LayerDesc(LayerKind.Concat, "route", ["up", "conv5"]))
    L.append(_conv("conv11", ch(128) + ch(256), ch(256), 3, 1, True, slope=slope))
    L.append(_conv("head2", ch(256), 255, 1, 0, False))
    spec = NetworkSpec(3, height, width, L)
    fill_random_weights(spec, seed)
    return spec


def make_small_spec(seed: int, in_channels: int, height: int, width: int) -> NetworkSpec:
    """make_small_spec, io.cpp:619-654."""
    spec = NetworkSpec(in_channels, height, width, [
        _conv("C1", in_channels, 16, 5, 2, True), _pool("P1"),
        _conv("C2", 16, 16, 3, 1, True), _conv("C3", 16, 8, 3, 1, False)])
    spec.layers[1].pool_size = spec.layers[1].pool_stride = 2
    fill_random_weights(spec, seed)
    return spec


class HostBuffer:
    """Pinned, mapped host memory (cbg_host_alloc) viewed as a numpy array."""

    def __init__(self, nbytes: int, dtype=np.uint8):
        p = C.c_void_p()
        check(lib.cbg_host_alloc(int(nbytes), C.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)
        itemsize = np.dtype(dtype).itemsize
        self.array = np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(self.ptr)).view(dtype)[
            :self.nbytes // itemsize]

    def __del__(self):
        if getattr(self, "ptr", None) and lib is not None:
            lib.cbg_host_free(C.c_void_p(self.ptr))
            self.ptr = None


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class Context:
    """One device + one CUDA stream (cbg_ctx)."""

    _default: Optional["Context"] = None

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.cbg_ctx_create(device, C.byref(h)))
        self.handle = h

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def synchronize(self):
        check(lib.cbg_ctx_sync(self.handle))

    def set_persistent_sms(self, sms: int):
        """SMs the persistent kernels of this context spread over (0 = all);
        for frames captured afterwards"""
        check(lib.cbg_ctx_set_persistent_sms(self.handle, int(sms)))

    @property
    def stream(self) -> int:
        return lib.cbg_ctx_stream(self.handle) or 0

    @property
    def copy_stream(self) -> int:
        """the copy-out stream of copy_output_detached (synchronize() waits for it too)"""
        return lib.cbg_ctx_copy_stream(self.handle) or 0

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.cbg_ctx_destroy(self.handle)
            self.handle = None


# ---------------------------------------------------------------------------
# layers
# ---------------------------------------------------------------------------
@dataclass
class UpstreamChange:
    """UpstreamChange, layers.hpp:16-19."""

    map: Optional[np.ndarray] = None
    indexes: Optional[np.ndarray] = None


@dataclass
class ConvForwardResult:
    """ConvForwardResult, layers.hpp:27-35."""

    out_map: np.ndarray
    indexes: np.ndarray
    eff_ops: int = 0
    worst_case_map: Optional[np.ndarray] = None
    propagated_px: int = -1


@dataclass
class PoolForwardResult:
    out_map: np.ndarray
    indexes: np.ndarray


def _f32(x, shape=None, what="input"):
    a = np.ascontiguousarray(x, dtype=np.float32)
    if shape is not None and a.shape != tuple(shape):
        raise InvalidInputError(f"{what}: shape {a.shape} != expected {tuple(shape)}")
    return a


def _up(up: Optional[UpstreamChange], h: int, w: int):
    if up is None:
        return None, None, 0
    m = None if up.map is None else np.ascontiguousarray(up.map, dtype=np.uint8)
    if m is not None and m.shape != (h, w):
        raise InvalidInputError("upstream map not in this layer's input frame")
    idx = None if up.indexes is None else np.ascontiguousarray(np.asarray(up.indexes, np.int32).reshape(-1, 2))
    return m, idx, (0 if idx is None else len(idx))


class CBConvLayer:
    """CBConvLayer, layers.hpp:45-69 / layers.cpp:33-131."""

    def __init__(self, spec: ConvSpec, tau: float, policy=DetectionPolicy.Detect, fuse_relu: bool = False,
                 mode=DetectMode.ClosedLoop, in_height: int = 0, in_width: int = 0, ctx: Context = None):
        self.ctx = ctx or Context.default()
        keep: list = []
        cs = spec._c(keep)
        h = C.c_void_p()
        check(lib.cbg_conv_create(self.ctx.handle, C.byref(cs), float(tau), int(policy), int(bool(fuse_relu)),
                                  int(mode), in_height, in_width, C.byref(h)))
        self.handle = h
        self.spec = spec
        self._tau = float(tau)
        self.policy = DetectionPolicy(policy)
        self.mode = DetectMode(mode)
        self.fuse_relu = bool(fuse_relu)
        self.in_h, self.in_w = in_height, in_width
        oh, ow = C.c_int(), C.c_int()
        check(lib.cbg_conv_out_dims(h, C.byref(oh), C.byref(ow)))
        self.out_h, self.out_w = oh.value, ow.value

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.cbg_conv_destroy(self.handle)
            self.handle = None

    @property
    def tau(self) -> float:
        return self._tau

    @tau.setter
    def tau(self, v: float):
        check(lib.cbg_conv_set_tau(self.handle, float(v)))
        self._tau = float(v)

    def ops_per_pixel(self) -> int:  # layers.hpp:65-67
        s = self.spec
        return 2 * s.out_channels * s.in_channels * s.kernel_h * s.kernel_w

    def dense_ops(self) -> int:
        return self.ops_per_pixel() * self.out_h * self.out_w

    def forward(self, x, upstream: Optional[UpstreamChange] = None, force_full_update: bool = False,
                record_worst_case: bool = False) -> ConvForwardResult:
        xa = _f32(x, (self.spec.in_channels, self.in_h, self.in_w), "CBConvLayer: input shape mismatch")
        m, idx, n = _up(upstream, self.in_h, self.in_w)
        flags = (_lib.FWD_FORCE_FULL if force_full_update else 0) | \
                (_lib.FWD_RECORD_WORST_CASE if record_worst_case else 0)
        eff = C.c_int64()
        check(lib.cbg_conv_forward(self.handle, fptr(xa), fptr(m), fptr(idx), n, flags, C.byref(eff)))
        out_map, indexes = self._changes()
        res = ConvForwardResult(out_map, indexes, eff.value)
        if record_worst_case:
            wm = np.zeros((self.out_h, self.out_w), np.uint8)
            cnt = C.c_int64()
            check(lib.cbg_conv_read_worst_case(self.handle, fptr(wm), C.byref(cnt)))
            res.worst_case_map, res.propagated_px = wm, cnt.value
        return res

    def _changes(self):
        m = np.zeros((self.out_h, self.out_w), np.uint8)
        rc = np.zeros((self.out_h * self.out_w, 2), np.int32)
        cnt = C.c_int64()
        check(lib.cbg_conv_read_changes(self.handle, fptr(m), fptr(rc), C.byref(cnt)))
        return m, rc[:cnt.value].copy()

    @property
    def prev_output(self) -> np.ndarray:
        y = np.empty((self.spec.out_channels, self.out_h, self.out_w), np.float32)
        check(lib.cbg_conv_read_output(self.handle, fptr(y)))
        return y

    @property
    def state(self) -> np.ndarray:
        y = np.empty((self.spec.in_channels, self.in_h, self.in_w), np.float32)
        check(lib.cbg_conv_read_state(self.handle, fptr(y)))
        return y


class CBPoolLayer:
    """CBPoolLayer, layers.hpp:78-91 / layers.cpp:133-179."""

    def __init__(self, size: int, stride: int, channels: int, in_height: int, in_width: int, out_height: int,
                 out_width: int, ctx: Context = None):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(lib.cbg_pool_create(self.ctx.handle, size, stride, channels, in_height, in_width, out_height,
                                  out_width, C.byref(h)))
        self.handle = h
        self.size, self.stride, self.channels = size, stride, channels
        self.in_h, self.in_w, self.out_h, self.out_w = in_height, in_width, out_height, out_width

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.cbg_pool_destroy(self.handle)
            self.handle = None

    def forward(self, x, upstream: Optional[UpstreamChange] = None,
                force_full_update: bool = False) -> PoolForwardResult:
        xa = _f32(x, (self.channels, self.in_h, self.in_w), "CBPoolLayer: input shape mismatch")
        m, idx, n = _up(upstream, self.in_h, self.in_w)
        check(lib.cbg_pool_forward(self.handle, fptr(xa), fptr(m), fptr(idx), n, int(bool(force_full_update))))
        m = np.zeros((self.out_h, self.out_w), np.uint8)
        rc = np.zeros((self.out_h * self.out_w, 2), np.int32)
        cnt = C.c_int64()
        check(lib.cbg_pool_read_changes(self.handle, fptr(m), fptr(rc), C.byref(cnt)))
        return PoolForwardResult(m, rc[:cnt.value].copy())

    @property
    def prev_output(self) -> np.ndarray:
        y = np.empty((self.channels, self.out_h, self.out_w), np.float32)
        check(lib.cbg_pool_read_output(self.handle, fptr(y)))
        return y


# ---------------------------------------------------------------------------
# network
# ---------------------------------------------------------------------------
@dataclass
class StatsConfig:  # network.hpp:91-96
    record_worst_case: bool = False
    record_maps: bool = False
    estimate_fg: bool = False
    timing: bool = False


@dataclass
class LayerFrameStats:  # network.hpp:98-110
    layer: str = ""
    changed_px: int = 0
    total_px: int = 0
    change_frac: float = 0.0
    eff_ops: int = 0
    wall_ns: int = 0
    propagated_px: int = -1
    fg_sp_ops: int = -1
    fg_fm_ops: int = -1
    map: Optional[np.ndarray] = None
    worst_case_map: Optional[np.ndarray] = None


@dataclass
class FrameStats:  # network.hpp:112-117
    frame: int = 0
    has_loss: bool = False
    loss: float = 0.0
    layers: List[LayerFrameStats] = field(default_factory=list)


@dataclass
class RunStats:  # network.hpp:119-126
    frames: List[FrameStats] = field(default_factory=list)

    def total_eff_ops(self, first_frame: int = 1) -> int:
        return sum(l.eff_ops for f in self.frames if f.frame >= first_frame for l in f.layers)

    def same_counts(self, other: "RunStats") -> bool:
        if len(self.frames) != len(other.frames):
            return False
        for a, b in zip(self.frames, other.frames):
            if a.frame != b.frame or a.has_loss != b.has_loss or a.loss != b.loss or len(a.layers) != len(b.layers):
                return False
            for x, y in zip(a.layers, b.layers):
                if (x.layer, x.changed_px, x.total_px, x.eff_ops, x.propagated_px) != \
                        (y.layer, y.changed_px, y.total_px, y.eff_ops, y.propagated_px):
                    return False
        return True


@dataclass
class NodeInfo:
    kind: LayerKind
    name: str
    inputs: List[int]
    out_shape: tuple
    in_shape: tuple
    policy: DetectionPolicy
    fuse_relu: bool
    tau: float
    ops_per_pixel: int


def validate_network(spec: NetworkSpec, taus: Sequence[float], policies=None, mode=DetectMode.ClosedLoop):
    """resolve() + convert_to_cb() checks on the host only (no device needed)."""
    keep: list = []
    cs = spec._c(keep)
    t = np.ascontiguousarray(taus, dtype=np.float32)
    p = None if policies is None else np.ascontiguousarray([int(x) for x in policies], dtype=np.int32)
    check(lib.cbg_net_validate(C.byref(cs), fptr(t), len(t), fptr(p), int(mode)))


class CBNetwork:
    """CBNetwork, network.hpp:141-173, for ``n_streams`` independent camera streams."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        n = C.c_int()
        check(lib.cbg_net_node_count(handle, C.byref(n)))
        check(lib.cbg_net_stream_count(handle, C.byref(C.c_int())))
        s = C.c_int()
        check(lib.cbg_net_stream_count(handle, C.byref(s)))
        self.n_streams = s.value
        self._nodes = []
        for i in range(n.value):
            info = _lib.NodeInfoC()
            check(lib.cbg_net_node_info(handle, i, C.byref(info)))
            self._nodes.append(NodeInfo(LayerKind(info.kind), info.name.decode(),
                                        list(info.inputs[:info.n_inputs]),
                                        (info.out_channels, info.out_height, info.out_width),
                                        (info.in_channels, info.in_height, info.in_width),
                                        DetectionPolicy(info.policy), bool(info.fuse_relu), info.tau,
                                        info.ops_per_pixel))
        self._frame_no = 0

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.cbg_net_destroy(self.handle)
            self.handle = None

    # -- structure --------------------------------------------------------
    def nodes(self) -> List[NodeInfo]:
        return self._nodes

    def input_shape(self):
        n0 = self._nodes[0]
        return n0.in_shape if n0.inputs and n0.inputs[0] < 0 else None

    def output_shape(self):
        return self._nodes[-1].out_shape

    def conv_layer_count(self) -> int:
        return sum(1 for n in self._nodes if n.kind == LayerKind.Conv)

    def thresholds(self) -> List[float]:
        t = np.zeros(max(1, self.conv_layer_count()), np.float32)
        check(lib.cbg_net_thresholds(self.handle, fptr(t), len(t)))
        return [float(v) for v in t[:self.conv_layer_count()]]

    def set_thresholds(self, taus: Sequence[float]):
        t = np.ascontiguousarray(taus, dtype=np.float32)
        check(lib.cbg_net_set_thresholds(self.handle, fptr(t), len(t)))

    def set_stream_thresholds(self, stream: int, taus: Sequence[float]):
        """Thresholds of one stream of the set (the others keep theirs)."""
        t = np.ascontiguousarray(taus, dtype=np.float32)
        check(lib.cbg_net_set_stream_thresholds(self.handle, stream, fptr(t), len(t)))

    def reset(self, stream: int = -1):
        check(lib.cbg_net_reset(self.handle, stream))

    def set_dense(self, dense: bool = True):
        check(lib.cbg_net_set_dense(self.handle, int(bool(dense))))

    def clone(self) -> "CBNetwork":
        h = C.c_void_p()
        check(lib.cbg_net_clone(self.handle, C.byref(h)))
        c = CBNetwork(h, self.ctx)
        c._frame_no = self._frame_no
        return c

    # -- frames -------------------------------------------------------------
    def enqueue(self, frames: np.ndarray, flags: int = 0):
        """Asynchronous forward of one frame per stream (frames: [S, C, H, W] or [C, H, W])."""
        check(lib.cbg_net_forward(self.handle, fptr(frames), flags))
        self._frame_no += 1

    def enqueue_device(self, device_ptr: int, flags: int = 0):
        """Forward with frames already in device memory (e.g. a torch CUDA tensor's data_ptr())."""
        check(lib.cbg_net_forward(self.handle, C.c_void_p(device_ptr), flags | _lib.FWD_INPUT_ON_DEVICE))
        self._frame_no += 1

    def enqueue_u8(self, frames_hwc: np.ndarray, flags: int = 0):
        """Asynchronous forward of 8-bit frames in PNM payload order ([S, H, W, C] uint8),
        converted on the device as load_pnm does (io.cpp:349-399: byte / 255.0f)."""
        fa = np.ascontiguousarray(frames_hwc, dtype=np.uint8)
        _, c, h, w = (self.n_streams,) + tuple(self._nodes[0].in_shape)
        if fa.size != self.n_streams * h * w * c:
            raise InvalidInputError("forward_u8: frame resolution mismatch")
        check(lib.cbg_net_forward_u8(self.handle, fa.ctypes.data_as(C.c_void_p), flags))
        self._frame_no += 1

    def enqueue_device_u8(self, device_ptr: int, flags: int = 0):
        """8-bit frames ([S, H, W, C] uint8) already in device memory."""
        check(lib.cbg_net_forward_u8(self.handle, C.c_void_p(device_ptr), flags | _lib.FWD_INPUT_ON_DEVICE))
        self._frame_no += 1

    def forward_frame_u8(self, frame_hwc, stream: int = 0) -> np.ndarray:
        """forward_frame on an 8-bit PNM-payload frame per stream ([S, H, W, C] or [H, W, C])."""
        self.enqueue_u8(frame_hwc)
        return self.output(stream)

    def forward_frame(self, frame, cfg: StatsConfig = None, frame_stats: Optional[FrameStats] = None,
                      stream: int = 0) -> np.ndarray:
        """forward_frame, network.cpp:309-414. ``frame`` holds one frame per stream
        ([S, C, H, W]; a single [C, H, W] frame is accepted when S == 1). Returns the
        last node's retained output of ``stream``."""
        cfg = cfg or StatsConfig()
        shp = self._nodes[0].in_shape
        fa = np.ascontiguousarray(frame, dtype=np.float32)
        want = (self.n_streams,) + tuple(shp)
        if fa.shape != want and not (self.n_streams == 1 and fa.shape == tuple(shp)):
            raise InvalidInputError("forward_frame: frame resolution mismatch")
        flags = _lib.FWD_RECORD_WORST_CASE if cfg.record_worst_case else 0
        self.enqueue(fa, flags)
        if frame_stats is not None:
            frame_stats.frame = self._frame_no
            frame_stats.layers = self.layer_stats(stream, cfg)
        return self.output(stream)

    def layer_stats(self, stream: int = 0, cfg: StatsConfig = None) -> List[LayerFrameStats]:
        cfg = cfg or StatsConfig()
        st = (_lib.LayerStatsC * len(self._nodes))()
        check(lib.cbg_net_read_stats(self.handle, stream, st, len(self._nodes)))
        rows = []
        for i, (n, s) in enumerate(zip(self._nodes, st)):
            row = LayerFrameStats(n.name, s.changed_px, s.total_px,
                                  s.changed_px / s.total_px if s.total_px else 0.0, s.eff_ops, 0,
                                  s.propagated_px)
            if cfg.record_maps:
                row.map = self.node_changes(i, stream)[0]
                if cfg.record_worst_case and n.kind == LayerKind.Conv:
                    row.worst_case_map = self.node_worst_case(i, stream)[0]
            rows.append(row)
        return rows

    def counts(self) -> np.ndarray:
        """changed_px of every node and stream of the last frame: [n_nodes, S]."""
        c = np.zeros((len(self._nodes), self.n_streams), np.int64)
        check(lib.cbg_net_read_counts(self.handle, fptr(c)))
        return c

    def output(self, stream: int = 0) -> np.ndarray:
        return self.node_output(-1, stream)

    def node_output(self, node: int, stream: int = 0) -> np.ndarray:
        shp = self._nodes[node].out_shape
        y = np.empty(shp, np.float32)
        check(lib.cbg_net_read_output(self.handle, node, stream, fptr(y)))
        return y

    def node_state(self, node: int, stream: int = 0) -> np.ndarray:
        y = np.empty(self._nodes[node].in_shape, np.float32)
        check(lib.cbg_net_read_state(self.handle, node, stream, fptr(y)))
        return y

    def node_changes(self, node: int, stream: int = 0):
        _, h, w = self._nodes[node].out_shape
        m = np.zeros((h, w), np.uint8)
        rc = np.zeros((h * w, 2), np.int32)
        cnt = C.c_int64()
        check(lib.cbg_net_read_changes(self.handle, node, stream, fptr(m), fptr(rc), C.byref(cnt)))
        return m, rc[:cnt.value].copy()

    def node_worst_case(self, node: int, stream: int = 0):
        _, h, w = self._nodes[node].out_shape
        m = np.zeros((h, w), np.uint8)
        cnt = C.c_int64()
        check(lib.cbg_net_read_worst_case(self.handle, node, stream, fptr(m), C.byref(cnt)))
        return m, cnt.value

    def set_kernel_timing(self, enabled: bool = True):
        check(lib.cbg_net_set_kernel_timing(self.handle, int(bool(enabled))))

    def timing_report(self) -> dict:
        import json
        buf = C.create_string_buffer(1 << 16)
        check(lib.cbg_net_timing_report(self.handle, buf, len(buf)))
        return json.loads(buf.value.decode())

    def output_bytes(self, node: int = -1) -> int:
        n = C.c_int64()
        check(lib.cbg_net_output_bytes(self.handle, node, C.byref(n)))
        return n.value

    def copy_output_async(self, host_ptr: int, node: int = -1):
        """Async D2H of a node's raw device output (NHWC, all streams) into pinned memory."""
        check(lib.cbg_net_copy_output_async(self.handle, node, C.c_void_p(host_ptr)))


    def copy_output_detached(self, host_ptr: int, node: int = -1):
        """copy_output_async through a device staging buffer, D2H on the context's
        copy-out stream: the next frame does not wait for PCIe (Context.synchronize waits for it)"""
        check(lib.cbg_net_copy_output_detached(self.handle, node, C.c_void_p(host_ptr)))
    def output_delta_bytes(self, node: int = -1) -> int:
        n = C.c_int64()
        check(lib.cbg_net_output_delta_bytes(self.handle, node, C.byref(n)))
        return n.value

    def copy_output_delta(self, host_ptr: int, node: int = -1):
        """this frame's changed pixels of `node` and their raw output vectors into
        pinned host memory (cbg_net_copy_output_delta layout: packed, only the
        changed bytes cross PCIe), on the context's copy-out stream"""
        check(lib.cbg_net_copy_output_delta(self.handle, node, C.c_void_p(host_ptr)))

    def last_delta_dma_bytes(self) -> int:
        n = C.c_int64()
        check(lib.cbg_net_last_delta_dma_bytes(self.handle, C.byref(n)))
        return n.value

    def apply_output_delta(self, host_ptr: int, mirror_ptr: int, node: int = -1, streams=None):
        """wait for the delta in host_ptr, scatter streams [s0, s1) into the host
        mirror of the raw output [S][H][W][Cs] (releases the GIL: callers may
        split the streams over threads)"""
        s0, s1 = streams if streams is not None else (0, self.n_streams)
        check(lib.cbg_net_apply_output_delta(self.handle, node, C.c_void_p(host_ptr), C.c_void_p(mirror_ptr),
                                             s0, s1))

    def delta_counts(self, host_buf: np.ndarray) -> np.ndarray:
        """per-stream changed-pixel counts at the head of a delta buffer"""
        return np.frombuffer(host_buf, np.int32, count=self.n_streams)

    def count_layout(self):
        """(slots, node->slot) of the device change-count array [S][slots]."""
        n = C.c_int()
        check(lib.cbg_net_count_slots(self.handle, C.byref(n)))
        slots = np.zeros(len(self._nodes), np.int32)
        check(lib.cbg_net_copy_counts_async(self.handle, None, fptr(slots)))
        return n.value, slots

    def kernel_labels(self, flags: int = 0):
        """labels of the kernels one frame launches, in launch order"""
        buf = C.create_string_buffer(1 << 16)
        check(lib.cbg_net_kernel_labels(self.handle, flags, buf, len(buf)))
        return json.loads(buf.value.decode())

    def detect_slots(self):
        """node -> slot of its detected (pre-dilation) input-pixel count in the
        count array (-1: not a detect-policy conv)."""
        slots = np.zeros(len(self._nodes), np.int32)
        check(lib.cbg_net_detect_slots(self.handle, fptr(slots)))
        return slots

    def copy_counts_async(self, host_ptr: int):
        check(lib.cbg_net_copy_counts_async(self.handle, C.c_void_p(host_ptr), None))

    def last_launches(self) -> int:
        n = C.c_int()
        check(lib.cbg_net_last_launches(self.handle, C.byref(n)))
        return n.value

    def synchronize(self):
        self.ctx.synchronize()


def convert_to_cb(spec: NetworkSpec, taus: Sequence[float], policies=None, mode=DetectMode.ClosedLoop,
                  n_streams: int = 1, ctx: Context = None) -> CBNetwork:
    """convert_to_cb, network.cpp:416-503 (the spec plays the DenseNetwork's role)."""
    ctx = ctx or Context.default()
    keep: list = []
    cs = spec._c(keep)
    t = np.ascontiguousarray(taus, dtype=np.float32)
    p = None if policies is None else np.ascontiguousarray([int(x) for x in policies], dtype=np.int32)
    h = C.c_void_p()
    check(lib.cbg_net_create(ctx.handle, C.byref(cs), fptr(t), len(t), fptr(p), int(mode), n_streams, C.byref(h)))
    return CBNetwork(h, ctx)


@dataclass
class SequenceResult:
    outputs: List[np.ndarray] = field(default_factory=list)
    stats: RunStats = field(default_factory=RunStats)


def loss_value(metric, pred: np.ndarray, ref: np.ndarray) -> float:
    """loss_value (calibration.cpp:51-53): mse (calibration.cpp:41-49) or
    1 - pixel_accuracy (argmax over channels, first maximum wins; a 1-channel
    reference holds class ids, calibration.cpp:26-39)."""
    pred = np.asarray(pred, np.float32)
    ref = np.asarray(ref, np.float32)
    if int(metric) == 0:
        if pred.shape != ref.shape:
            raise InvalidInputError("mse: shapes differ")
        return float(np.mean((pred.astype(np.float64) - ref.astype(np.float64)) ** 2))
    if pred.shape[1:] != ref.shape[1:]:
        raise InvalidInputError("pixel_accuracy: spatial dims differ")
    if ref.shape[0] != 1 and ref.shape[0] != pred.shape[0]:
        raise InvalidInputError("pixel_accuracy: reference channels must be 1 (labels) or match")
    a = np.argmax(pred, axis=0)  # numpy argmax returns the first maximum, as argmax_channel
    r = ref[0].astype(np.int64) if ref.shape[0] == 1 else np.argmax(ref, axis=0)
    return 1.0 - float(np.mean(a == r))


def forward_sequence(net: CBNetwork, frames, reference=None, metric=0, cfg: StatsConfig = None) -> SequenceResult:
    """forward_sequence, network.cpp:505-525 (per-frame loss under `metric` when a reference is given)."""
    if reference is not None and len(reference) != len(frames):
        raise InvalidInputError("forward_sequence: reference count != frame count")
    res = SequenceResult()
    for t, f in enumerate(frames):
        fs = FrameStats(frame=t + 1)
        out = net.forward_frame(f, cfg, fs)
        fs.frame = t + 1
        if reference is not None:
            fs.loss = loss_value(metric, out, reference[t])
            fs.has_loss = True
        res.outputs.append(out)
        res.stats.frames.append(fs)
    return res


def write_stats_csv(run: RunStats) -> str:
    """write_stats_csv (io.cpp:660-672): the same columns and number formats
    (change_frac "%.6f", loss "%.9g")."""
    out = ["frame,layer,changed_px,change_frac,eff_ops,wall_ns,loss\n"]
    for f in run.frames:
        for l in f.layers:
            out.append(f"{f.frame},{l.layer},{l.changed_px},{l.change_frac:.6f},{l.eff_ops},{l.wall_ns},"
                       + (f"{f.loss:.9g}" if f.has_loss else "") + "\n")
    return "".join(out)
