/*
 * cbg.h — C ABI of the B200-native change-based inference (CBinfer) hot path.
 *
 * This is the drop-in boundary for the reference's layer/operator API
 * (reference: /root/reference/proj, namespace cbi). Every entry point below
 * replaces one reference interface; the citation names the reference
 * file:line it mirrors. Plain pointers and sizes only: no C++ or torch types
 * cross this boundary.
 *
 * Conventions
 *  - Every function returns an int status: CBG_OK (0) or one of the error
 *    categories below. The matching message is available from
 *    cbg_last_error() (thread-local), and the C++ wrapper
 *    (include/cbg/cbi_gpu.hpp) rethrows it as the matching cbi-style
 *    exception: INVALID_INPUT -> InvalidInputError, CONFIG -> ConfigError
 *    (reference: proj/include/cbi/common.hpp:11-21).
 *  - Tensors crossing the boundary on the host side use the reference's
 *    Tensor3 layout: channel-major, row-major planes, fp32
 *    (reference: proj/include/cbi/tensor.hpp:13-35).
 *  - Index lists cross as int32 (row, col) pairs in row-major order
 *    (reference: PixelIndex/IndexList, tensor.hpp:38-44).
 *  - All device work is enqueued on the context's CUDA stream. Only the
 *    cbg_*_read_* functions and cbg_ctx_sync synchronise.
 *  - A handle must be used by one host thread at a time (the reference's
 *    layers are externally serialised as well). Distinct
 *    handles may be used concurrently.
 */
#ifndef CBG_H_
#define CBG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBG_ABI_VERSION 1

/* ---- status codes (reference error taxonomy, common.hpp:11-48) ---------- */
enum {
  CBG_OK = 0,
  CBG_ERR_INVALID_INPUT = 1, /* cbi::InvalidInputError */
  CBG_ERR_CONFIG = 2,        /* cbi::ConfigError */
  CBG_ERR_CUDA = 3,          /* CUDA runtime / launch failure */
  CBG_ERR_OOM = 4,           /* device allocation failure */
  CBG_ERR_UNSUPPORTED = 5    /* no sm_100 device, or a shape the kernels do not cover */
};

/* ---- enums mirroring the reference ---------------------------------------- */
/* LayerKind, network.hpp:10 */
enum { CBG_LAYER_CONV = 0, CBG_LAYER_ACT = 1, CBG_LAYER_POOL = 2, CBG_LAYER_ADD = 3, CBG_LAYER_CONCAT = 4,
       /* extension beyond the reference (network.hpp:10 has no upsample): nearest-neighbour
        * upsampling by an integer factor (YOLOv3-style detectors) */
       CBG_LAYER_UPSAMPLE = 5 };
/* DetectionPolicy, layers.hpp:8 */
enum { CBG_POLICY_DETECT = 0, CBG_POLICY_PROPAGATE = 1, CBG_POLICY_REUSE1X1 = 2 };
/* DetectMode, change.hpp:34 */
enum { CBG_MODE_FEEDFORWARD = 0, CBG_MODE_CLOSEDLOOP = 1 };

/* forward flags (ConvForwardOptions, layers.hpp:21-25) */
enum {
  CBG_FWD_FORCE_FULL = 1u << 0,        /* force_full_update: bootstrap-style full recompute */
  CBG_FWD_RECORD_WORST_CASE = 1u << 1, /* record_worst_case: also compute propagate_changes(up) */
  CBG_FWD_INPUT_ON_DEVICE = 1u << 2,   /* the frame pointer is a device pointer */
  CBG_FWD_BROADCAST_INPUT = 1u << 3    /* one frame [C][H][W] is fed to every stream (fp32 API) */
};

/* ---- descriptions --------------------------------------------------------- */
/* ConvSpec, tensor.hpp:54-80. weights: [out][in][kh][kw] fp32, bias: [out]. */
typedef struct cbg_conv_spec {
  int in_channels, out_channels;
  int kernel_h, kernel_w;
  int stride, padding;
  int out_h, out_w; /* 0 = derived floor formula; >0 pins (crop), tensor.hpp:49-53 */
  const float* weights;
  const float* bias;
} cbg_conv_spec;

/* LayerDesc, network.hpp:25-37 */
typedef struct cbg_layer_desc {
  int kind;                /* CBG_LAYER_* */
  const char* name;        /* NULL or "" -> "L<i+1>" (network.cpp:14-16) */
  int n_from;              /* 0 -> previous row (network input for row 0) */
  const char* const* from; /* producer names; "input" = network input */
  cbg_conv_spec conv;      /* CONV */
  int fuse_relu;           /* CONV */
  int pool_size, pool_stride, pool_out_h, pool_out_w; /* POOL (out dims 0 = floor formula) */
  /* Extensions beyond the reference (parity checked against the test-side C
   * restatement oracle/cbi_oracle.c only: "parity unpinned"):
   *   act_slope: ACT rows, and CONV rows with fuse_relu — 0 = ReLU
   *              (std::max(v, 0.f), the reference), > 0 = leaky ReLU
   *              v < 0 ? v * act_slope : v (Darknet's leaky, slope 0.1);
   *   upsample:  UPSAMPLE rows, the integer factor: out(j, i) = in(j / f, i / f),
 *              out dims in * f, or pool_out_h / pool_out_w when > 0 (a crop). */
  float act_slope;
  int upsample;
} cbg_layer_desc;

/* NetworkSpec, network.hpp:39-44 */
typedef struct cbg_network_spec {
  int in_channels, in_height, in_width;
  int n_layers;
  const cbg_layer_desc* layers;
} cbg_network_spec;

/* SyntheticConfig, io.hpp:47-58 */
typedef struct cbg_synthetic_config {
  int height, width, channels, n_frames;
  int n_objects, object_size;
  int velocity_y, velocity_x;
  float noise_std;
  uint32_t seed;
} cbg_synthetic_config;

/* Per-node static information (CBNode, network.hpp:129-137). */
typedef struct cbg_node_info {
  int kind;           /* CBG_LAYER_* (never ACT: absorbed) */
  char name[64];
  int n_inputs;
  int inputs[8];      /* node ids, -1 = network input */
  int out_channels, out_height, out_width;
  int in_channels, in_height, in_width;
  int policy;         /* conv only */
  int fuse_relu;      /* conv only */
  float tau;          /* conv only */
  int64_t ops_per_pixel; /* conv only: 2*Cout*Cin*kh*kw (layers.hpp:65-67) */
} cbg_node_info;

/* LayerFrameStats subset (network.hpp:98-110), deterministic fields only. */
typedef struct cbg_layer_stats {
  int64_t changed_px;
  int64_t total_px;
  int64_t eff_ops;
  int64_t propagated_px; /* -1 = not recorded */
} cbg_layer_stats;

typedef struct cbg_ctx_s* cbg_ctx;
typedef struct cbg_net_s* cbg_net;
typedef struct cbg_conv_s* cbg_conv;
typedef struct cbg_pool_s* cbg_pool;

/* ---- errors / library ------------------------------------------------------ */
const char* cbg_last_error(void);
int cbg_abi_version(void);
/* 1 when a CUDA device of compute capability 10.x is visible. */
int cbg_device_available(void);

/* ---- context: one device + one CUDA stream -------------------------------- */
int cbg_ctx_create(int device, cbg_ctx* out);
void cbg_ctx_destroy(cbg_ctx ctx);
/* Waits for the ctx stream and the copy-out stream (cbg_net_copy_output_detached). */
int cbg_ctx_sync(cbg_ctx ctx);
/* The context's cudaStream_t, for interop (returned as void*). */
void* cbg_ctx_stream(cbg_ctx ctx);
/* SMs the persistent tcgen05 GEMMs of this context spread over; 0 = all (default). With several contexts' stream sets in
 * flight at once, a share of the GPU per GEMM lets the sets' GEMMs and their
 * memory-bound kernels run side by side (bench.py: a third of the SMs for 4
 * sets). Applies to frames captured after the call (set it before the first). */
int cbg_ctx_set_persistent_sms(cbg_ctx ctx, int sms);

/* ---- host-side harness mirrors of the reference io.cpp (no device) -------- */
/* gen_synthetic, io.cpp:499-552: frames_out holds n_frames*channels*height*width
 * floats (CHW per frame); corners_out (nullable) n_frames*n_objects*2 ints. */
int cbg_gen_synthetic(const cbg_synthetic_config* cfg, float* frames_out, int32_t* corners_out);
/* fill_random_weights, io.cpp:554-566: conv rows in spec order; weights[i]
 * and biases[i] are writable buffers for the i-th CONV row. */
int cbg_fill_random_weights(const cbg_network_spec* spec, uint32_t seed, float* const* weights,
                            float* const* biases);

/* ---- network (CBNetwork, network.hpp:141-181) ----------------------------- */
/* resolve() + convert_to_cb() validation only, no device (network.cpp:37-133,416-503). */
int cbg_net_validate(const cbg_network_spec* spec, const float* taus, int n_taus,
                     const int* policies /* nullable */, int mode);
/* convert_to_cb(DenseNetwork(spec), taus, policies, mode) for n_streams
 * independent camera streams (each one CBNetwork instance of the reference;
 * they share the immutable weights and are processed in the same launches). */
int cbg_net_create(cbg_ctx ctx, const cbg_network_spec* spec, const float* taus, int n_taus,
                   const int* policies /* nullable */, int mode, int n_streams, cbg_net* out);
void cbg_net_destroy(cbg_net net);
/* Copying a CBNetwork yields independent streams (network.hpp:139-141). */
int cbg_net_clone(cbg_net net, cbg_net* out);
int cbg_net_node_count(cbg_net net, int* n_nodes);
int cbg_net_stream_count(cbg_net net, int* n_streams);
int cbg_net_node_info(cbg_net net, int node, cbg_node_info* info);
/* forward_frame (network.cpp:309-414) for every stream at once: frames holds
 * n_streams frames, CHW each. Host pointers are copied in on the ctx stream
 * (pinned memory makes it asynchronous). Flags: CBG_FWD_*. */
int cbg_net_forward(cbg_net net, const float* frames, unsigned flags);
/* Same frame step with 8-bit frames in the byte order of a binary PNM payload
 * (P5 gray / P6 RGB: [n_streams][H][W][C] interleaved, maxval 255), converted
 * on the device exactly as load_pnm does (io.cpp:349-399: planar fp32 =
 * byte / 255.0f, IEEE division). A quarter of the fp32 ingest bytes. The
 * network input must have C <= 4 channels. Flags: CBG_FWD_*. */
int cbg_net_forward_u8(cbg_net net, const uint8_t* frames_hwc, unsigned flags);
/* reset() (network.cpp:274-290); stream = -1 resets all streams. */
int cbg_net_reset(cbg_net net, int stream);
/* set_thresholds() / thresholds() (network.cpp:256-272). */
int cbg_net_set_thresholds(cbg_net net, const float* taus, int n_taus);
int cbg_net_thresholds(cbg_net net, float* taus, int n_taus);
/* Thresholds of one stream only (the others keep theirs): a stream set can
 * evaluate several threshold vectors at once (GPU calibration, below). */
int cbg_net_set_stream_thresholds(cbg_net net, int stream, const float* taus, int n_taus);
/* Dense path: every frame is a full update through the same kernels and
 * GEMM precision (the implementation's own dense-conv baseline). */
int cbg_net_set_dense(cbg_net net, int dense);

/* ---- synchronising readers ----------------------------------------------- */
/* Node retained output (node = -1 -> last node, network.cpp:307), CHW. */
int cbg_net_read_output(cbg_net net, int node, int stream, float* out_chw);
/* Detect-policy input state (InputState, change.hpp:30-32), CHW. */
int cbg_net_read_state(cbg_net net, int node, int stream, float* out_chw);
/* Last frame's output-frame change map (uint8 0/1, H*W) and index list. */
int cbg_net_read_changes(cbg_net net, int node, int stream, uint8_t* map_out /* nullable */,
                         int32_t* rowcol_out /* nullable, 2*count */, int64_t* count_out);
/* Last frame's worst-case map (record_worst_case), conv nodes only. */
int cbg_net_read_worst_case(cbg_net net, int node, int stream, uint8_t* map_out,
                            int64_t* count_out);
/* Per-node stats of the last frame, stats[node] for one stream. */
int cbg_net_read_stats(cbg_net net, int stream, cbg_layer_stats* stats, int n_nodes);
/* changed_px of every node and stream of the last frame: counts[node*S+s]. */
int cbg_net_read_counts(cbg_net net, int64_t* counts);

/* ---- standalone layers (CBConvLayer / CBPoolLayer, layers.hpp:45-91) ------- */
/* CBConvLayer ctor, layers.cpp:33-53. */
int cbg_conv_create(cbg_ctx ctx, const cbg_conv_spec* spec, float tau, int policy, int fuse_relu,
                    int mode, int in_h, int in_w, cbg_conv* out);
void cbg_conv_destroy(cbg_conv layer);
int cbg_conv_out_dims(cbg_conv layer, int* out_h, int* out_w);
/* CBConvLayer::forward, layers.cpp:55-131. x: host CHW [in_c][in_h][in_w];
 * up_map: nullable host uint8 [in_h][in_w] (the UpstreamChange map);
 * up_rowcol: nullable host int32 pairs (UpstreamChange indexes, in the
 * upstream frame). eff_ops_out: nullable. Flags: CBG_FWD_FORCE_FULL,
 * CBG_FWD_RECORD_WORST_CASE. */
int cbg_conv_forward(cbg_conv layer, const float* x, const uint8_t* up_map,
                     const int32_t* up_rowcol, int64_t up_count, unsigned flags,
                     int64_t* eff_ops_out);
int cbg_conv_read_output(cbg_conv layer, float* out_chw);
int cbg_conv_read_state(cbg_conv layer, float* out_chw);
int cbg_conv_read_changes(cbg_conv layer, uint8_t* map_out, int32_t* rowcol_out,
                          int64_t* count_out);
int cbg_conv_read_worst_case(cbg_conv layer, uint8_t* map_out, int64_t* count_out);
int cbg_conv_set_tau(cbg_conv layer, float tau);

/* CBPoolLayer ctor, layers.cpp:133-146. */
int cbg_pool_create(cbg_ctx ctx, int size, int stride, int channels, int in_h, int in_w,
                    int out_h, int out_w, cbg_pool* out);
void cbg_pool_destroy(cbg_pool layer);
/* CBPoolLayer::forward, layers.cpp:148-179. */
int cbg_pool_forward(cbg_pool layer, const float* x, const uint8_t* up_map,
                     const int32_t* up_rowcol, int64_t up_count, int force_full_update);
int cbg_pool_read_output(cbg_pool layer, float* out_chw);
int cbg_pool_read_changes(cbg_pool layer, uint8_t* map_out, int32_t* rowcol_out,
                          int64_t* count_out);

/* ---- threshold calibration on the GPU (calibration.hpp:16-84) -------------- */
/* An evaluation sequence (EvalSequence, calibration.hpp:19-22): host frames
 * [n_frames][C][H][W] (network input) and one reference output per frame,
 * [n_frames][ref_channels][Ho][Wo] (ref_channels = the net's output channels,
 * or 1 = class labels for the pixel-accuracy metric). */
typedef struct cbg_eval_sequence {
  int n_frames;
  const float* frames;
  const float* references;
  int ref_channels;
} cbg_eval_sequence;

enum { CBG_LOSS_MSE = 0, CBG_LOSS_PIXEL_ACCURACY_DELTA = 1 };  /* LossMetric, network.hpp:183 */
enum { CBG_AGG_MEAN = 0, CBG_AGG_WORST = 1 };                   /* LossAggregation, calibration.hpp:26 */

/* CalibConfig, calibration.hpp:28-36 (budget_overrides nullable). */
typedef struct cbg_calib_config {
  double initial_tau;
  double growth_factor;
  double per_layer_budget;
  const double* budget_overrides;
  int n_budget_overrides;
  int metric;
  int aggregation;
  int max_steps;
} cbg_calib_config;

typedef struct cbg_calib_trace_point {  /* CalibTracePoint, calibration.hpp:38-42 */
  int layer;
  double tau;
  double loss;
} cbg_calib_trace_point;

/* select_thresholds (calibration.cpp:95-141) with the replays on the GPU: for
 * each conv layer, the base vector and all max_steps geometric candidates are
 * replayed at once as the streams of one stream set per sequence, and the
 * reference's sequential rule (keep the last candidate before the first budget
 * violation) is applied to the losses. `proto` supplies topology, policies and
 * mode (its thresholds and state are not used). taus_out / hit_cap_out: one per
 * conv layer; trace_out (nullable) gets the reference's trace, trace_len its
 * length (capped at trace_cap). */
int cbg_select_thresholds(cbg_net proto, const cbg_eval_sequence* seqs, int n_seqs, const cbg_calib_config* cfg,
                          float* taus_out, uint8_t* hit_cap_out, cbg_calib_trace_point* trace_out, int trace_cap,
                          int* trace_len);

typedef struct cbg_tradeoff_row {  /* TradeoffRow, calibration.hpp:56-61 */
  double factor;
  double loss;
  int64_t total_eff_ops;
  int64_t wall_ns;
} cbg_tradeoff_row;

/* sweep_threshold_factor (calibration.cpp:143-180): every factor's scaled
 * vector replayed from reset as one stream per factor; loss = mean per-frame
 * loss and ops = conv-op total over post-bootstrap frames. wall_ns = device
 * time of the replay shared by all factors of a sequence, split evenly. */
int cbg_sweep_threshold_factor(cbg_net proto, const float* base_tau, int n_tau, const double* factors,
                               int n_factors, const cbg_eval_sequence* seqs, int n_seqs, int metric,
                               cbg_tradeoff_row* rows_out);

/* ---- instrumentation / async I/O (bench, profiling) ----------------------- */
/* Kernel launches enqueued per cbg_net_forward (one frame of every stream). */
int cbg_net_last_launches(cbg_net net, int* launches);
/* Per-kernel CUDA-event timing: while enabled, forwards launch eagerly with an
 * event pair around every kernel; the report is a JSON object
 * {"frames": F, "kernels": {"<node>.<kernel>": [total_ms, launches], ...}}.
 * Enabling (or disabling) clears the accumulators. */
int cbg_net_set_kernel_timing(cbg_net net, int enabled);
int cbg_net_timing_report(cbg_net net, char* buf, int len);
/* Asynchronous D2H copy of a node's retained output in the device layout
 * (NHWC fp32, channel stride round_up(C,4), all streams) on the ctx stream. */
int cbg_net_copy_output_async(cbg_net net, int node, void* host_dst);
/* The same bytes, pipelined for serving: a device-to-device copy into one of
 * two staging buffers on the ctx stream, then the D2H on the context's
 * copy-out stream (cbg_ctx_copy_stream), so the next frame's kernels do not
 * wait for PCIe. Complete after cbg_ctx_sync (which waits for both streams)
 * or after the copy-out stream. host_dst should be pinned. */
int cbg_net_copy_output_detached(cbg_net net, int node, void* host_dst);
void* cbg_ctx_copy_stream(cbg_ctx ctx);
/* Delta output, the reference's full-output semantics (forward_frame returns
 * the whole retained output, network.cpp:412-413) with only this frame's
 * changes crossing PCIe: after a frame, the node's changed pixels and their raw
 * output vectors [Cs floats, the layout of cbg_net_copy_output_async] are
 * packed on the ctx stream and copied into host_buf (pinned, mapped host
 * memory of cbg_net_output_delta_bytes) on the copy-out stream:
 *   int32 n[S] (padded to 16 B), then per stream: int32 ids[n_s] (padded to
 *   16 B), float vals[n_s][Cs]. cbg_net_apply_output_delta
 * waits for the copy into host_buf, then scatters streams [stream_begin,
 * stream_end) into a host mirror [S][H][W][Cs] of the raw output that the
 * caller keeps across frames (initialised from a full copy, or zeros before the
 * first frame: every pixel of a full update is in the delta). The apply may run
 * on another host thread while the net's frame and copy calls go on, as long
 * as host_buf is not handed to a new copy before its apply returned. */
int cbg_net_output_delta_bytes(cbg_net net, int node, int64_t* bytes);
/* Pinned, mapped, portable host memory (what the copy functions above expect). */
int cbg_host_alloc(int64_t bytes, void** ptr);
void cbg_host_free(void* ptr);
int cbg_net_copy_output_delta(cbg_net net, int node, void* host_buf);
/* Bytes the last cbg_net_copy_output_delta moved by DMA (an estimate from the
 * recently applied deltas + 25%; a larger delta's remaining bytes are written
 * by an overflow kernel). */
int cbg_net_last_delta_dma_bytes(cbg_net net, int64_t* bytes);
int cbg_net_apply_output_delta(cbg_net net, int node, const void* host_buf, float* mirror, int stream_begin,
                               int stream_end);
int cbg_net_output_bytes(cbg_net net, int node, int64_t* bytes);
/* Asynchronous D2H copy of the per-frame change counts [n_streams][slots]
 * (int32, slots = cbg_net_count_slots) into host memory; node_slot (nullable)
 * receives each node's slot. */
int cbg_net_copy_counts_async(cbg_net net, int32_t* host_dst, int32_t* node_slot);
int cbg_net_count_slots(cbg_net net, int* slots);
/* Slot (in the same count array) of each node's detected input pixels before
 * dilation (the detect map of a detect-policy conv, change.cpp:20-43), -1 for
 * other nodes. Not a reference interface: the reference keeps this map
 * internal to CBConvLayer::forward (layers.cpp:74-86); it is the paper's
 * "changed pixels" of the input. */
int cbg_net_detect_slots(cbg_net net, int32_t* det_slot);
/* Labels ("<node>.<kernel>") of the kernels one frame launches with these
 * forward flags, in launch order, as a JSON list (instrumentation: matches
 * the timing report and ncu launch lists). */
int cbg_net_kernel_labels(cbg_net net, unsigned flags, char* buf, int len);
/* Debug builds only (-DCBG_TRACE, libcbg_trace.so): per-K-block clock64 timeline
 * of CTA 0 of the last GEMM launch, [6][4096]; returns entries copied (0 when
 * tracing is compiled out). */
int cbg_debug_gemm_trace(unsigned long long* buf, int n);

#ifdef __cplusplus
}
#endif
#endif /* CBG_H_ */
