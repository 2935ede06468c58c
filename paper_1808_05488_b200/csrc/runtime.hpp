// runtime.hpp — host runtime of the B200 CBinfer path.
//
// Mirrors the reference network layer (network.hpp:91-195) with device-resident,
// multi-stream state:
//   * Topology   = resolve() + convert_to_cb() (network.cpp:37-133, 416-503),
//                  host-only, same rules and error categories.
//   * Net        = CBNetwork for S independent camera streams that share the
//                  immutable weights; one launch per kernel step covers every
//                  stream (grid.y = stream), one CUDA graph per frame.
//   * standalone CBConvLayer / CBPoolLayer are a Net whose producer is an
//     "external" node fed from host buffers (layers.hpp:45-91).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cbg.h"
#include "kernels.hpp"

namespace cbg {

// Error carrying a cbg status code (cbi::InvalidInputError / ConfigError / ...).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void throw_invalid(const std::string& m);
[[noreturn]] void throw_config(const std::string& m);
void cuda_check(cudaError_t e, const char* what);

struct ConvDesc {
  int in_channels = 0, out_channels = 0, kernel_h = 0, kernel_w = 0, stride = 1, padding = 0;
  int out_h = 0, out_w = 0;
  std::vector<float> weights, bias;
};
int conv_out_dim(int in_dim, int kernel, int stride, int padding, int pinned);  // tensor.cpp:9-28
void validate_conv(const ConvDesc& c);                                          // tensor.cpp:30-43
ConvDesc conv_from_c(const cbg_conv_spec& s);

// One CB node after conversion (CBNode, network.hpp:129-137).
struct NodeDesc {
  int kind = CBG_LAYER_CONV;  // CONV / POOL / ADD / CONCAT, or kExternal
  std::string name;
  std::vector<int> inputs;    // node ids, -1 = network input
  int C = 0, H = 0, W = 0;    // out shape
  int Ci = 0, Hi = 0, Wi = 0; // shape of inputs[0]
  ConvDesc conv;
  float tau = 0.0f;
  int policy = CBG_POLICY_DETECT;
  bool relu = false;
  float slope = 0.0f;         // fused activation: 0 = ReLU (the reference), > 0 = leaky ReLU (extension)
  int pool_size = 0, pool_stride = 0;
  int up = 0;                 // CBG_LAYER_UPSAMPLE factor (extension)
};
constexpr int kExternal = -100;

struct Topology {
  int C = 0, H = 0, W = 0;  // network input
  int mode = CBG_MODE_CLOSEDLOOP;
  std::vector<NodeDesc> nodes;
};
// resolve + convert_to_cb, throwing Error with the reference's categories.
Topology convert(const cbg_network_spec& spec, const float* taus, int n_taus, const int* policies, int mode);

// ---- device resources ---------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept;
  ~DevBuf();
  void alloc(size_t n);  // zero-initialised
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  // SMs the persistent tcgen05 GEMMs of this context spread over (0 = all):
  // with several contexts' stream sets in flight, a share of the GPU per GEMM
  // lets their GEMMs and the memory-bound kernels run side by side instead of
  // queueing for every SM
  int persistent_sms = 0;
  int persistent() const { return persistent_sms > 0 && persistent_sms < sm_count ? persistent_sms : sm_count; }
  cudaStream_t stream = nullptr;
  cudaStream_t d2h = nullptr;  // copy-out stream of the detached output copies (cbg_ctx_sync waits for both)
  explicit Ctx(int dev);
  ~Ctx();
};

struct NodeRT {
  NodeDesc d;
  int Cs = 0, Csi = 0;           // padded channel strides (out / in)
  // conv
  int npad = 0, n_tiles = 0, KB = 0;
  int prec = 1;                  // tcgen05 operand split: 0 = 3xTF32, 1 = 3xFP16 (scaled)
  bool tma_a = false;            // 1x1 layer, staged A path fed by TMA gather4 (CBG_TMA_1X1=1, experiment)
  CUtensorMap tmap{};
  const float* tmap_src = nullptr;
  int w_exp = 0;                 // fp16: weights scaled by 2^-w_exp in the image
  bool exact = false;            // CUDA-core bit-exact path (conv_exact.cu) instead of tcgen05
  bool state_chw = false;        // first-layer exact conv: input state as CHW planes (= the frame layout)
  DevBuf wimg, ktab, bias, wraw; // wraw: [Cout][Cin*kh*kw] fp32 for the exact path
  DevBuf state;                  // Detect policy
  uint32_t* inmap = nullptr;     // Detect policy: bitmap of detected input pixels [S][Hi][nw] (in Net::clear_)
  size_t inmap_words = 0;
  bool inmap_plain = false;      // first detect: words merged in registers (DetectFrameArgs::map_plain)
  DevBuf state8;                 // first layer, 8-bit ingest: byte shadow of the state (DetectFrameArgs::state8)
  DevBuf split, split_e;         // 3xFP16 GEMM input: pre-split copy of the state (DetectListArgs::split)
  // every node
  DevBuf out;                    // [S][H][W][Cs]
  DevBuf outmap_own, idx_own;    // output bitmap [S][H][nw] and index list [S][H*W]
  uint32_t* outmap = nullptr;    // may alias the producer (Reuse1x1)
  int32_t* idx = nullptr;
  int count_slot = 0;            // index into Net::counts ([slot][S]): output list length
  int det_slot = -1;             // Detect policy: detected (pre-dilation) input pixels
  DilateCompactArgs dc{};        // geometry of this node's compaction (rows, bands, warps, smem)
  int pool_child = -1;           // 2x2/2 pool whose map and list this node's compaction also derives
  int fused_into = -1;           // pool: the producer whose compaction derives its map and list
  // worst-case map (record_worst_case)
  DevBuf wc_map, wc_idx;
  int wc_slot = -1;
  DilateCompactArgs dc_wc{};
};

class Net {
 public:
  Net(Ctx* ctx, Topology topo, int n_streams);
  ~Net();
  Net(const Net&) = delete;
  Net& operator=(const Net&) = delete;
  std::unique_ptr<Net> clone() const;

  int streams() const { return S_; }
  const Topology& topology() const { return topo_; }
  const std::vector<NodeRT>& nodes() const { return nodes_; }

  void forward(const float* frames, unsigned flags);
  void forward_u8(const uint8_t* frames_hwc, unsigned flags);  // PNM-payload frames (load_pnm semantics)
  // standalone layers: external producer contents (node 0 must be kExternal)
  void set_external(const float* x_chw, const uint8_t* map, const int32_t* rowcol, int64_t n, bool full = false);
  void reset(int stream);
  void set_thresholds(const std::vector<float>& taus);
  void set_stream_thresholds(int stream, const std::vector<float>& taus);  // one stream's thresholds
  std::vector<float> thresholds() const;
  void set_dense(bool dense);

  void read_output(int node, int stream, float* out_chw);
  void read_state(int node, int stream, float* out_chw);
  void read_changes(int node, int stream, uint8_t* map, int32_t* rowcol, int64_t* count, bool worst = false);
  void read_counts(std::vector<int32_t>& counts);  // [S][count_slots()]
  int64_t count_of(const std::vector<int32_t>& counts, int node, int stream, bool worst = false) const;
  bool has_worst_case(int node) const { return nodes_[node].wc_slot >= 0 && last_flags_ & CBG_FWD_RECORD_WORST_CASE; }

  int last_launches() const { return last_launches_; }
  // Per-kernel CUDA-event timing (eager launches, one sync per frame): label
  // "<node>.<kernel>" -> accumulated ms and launch count. Instrumentation only.
  void set_timing(bool on);
  std::string timing_report() const;  // JSON object
  // labels of the kernels one frame launches, in launch order (no launches)
  std::vector<std::string> kernel_labels(unsigned flags);
  void copy_output_async(int node, void* host_dst);  // raw NHWC [S][H][W][Cs] on the ctx stream
  // the same bytes through a device staging buffer: D2D on the ctx stream, D2H
  // on the ctx's copy-out stream, so the next frame does not wait for PCIe
  void copy_output_detached(int node, void* host_dst);
  void copy_counts_async(int32_t* host_dst);         // [S][count_slots()] on the ctx stream
  // Delta output (kernels.hpp DeltaArgs layout): the node's changed pixels of
  // this frame and their raw output vectors, packed on the ctx stream, then on
  // the copy-out stream a DMA of an estimated prefix (the recent sizes + 25%)
  // and an overflow kernel that writes any bytes past it into the pinned
  // (mapped) host buffer; apply_output_delta waits for that copy and scatters
  // streams [s0, s1) into a host mirror of the raw output [S][H][W][Cs].
  size_t output_delta_bytes(int node) const;
  void copy_output_delta(int node, void* host_buf);
  void apply_output_delta(int node, const void* host_buf, float* mirror, int s0, int s1);
  size_t last_delta_dma_bytes() const { return delta_dma_last_; }  // DMA size of the last copy_output_delta
  int count_slots() const { return cnt_stride_; }  // counters per stream in the [S][slots] count array
  int node_slot(int node) const { return nodes_[node].count_slot; }
  int det_slot(int node) const { return nodes_[node].det_slot; }

 private:
  void build();
  // kernels of one frame (graph body); slot8 = which 8-bit ingest pointer slot the first detect reads;
  // s8 = the first detect compares against the 8-bit state shadow
  void enqueue_frame(unsigned flags, bool u8 = false, bool bcast = false, int slot8 = 0, bool s8 = false);
  int launch_count(unsigned flags) const;

  Ctx* ctx_;
  Topology topo_;
  int S_;
  std::vector<NodeRT> nodes_;
  DevBuf frame_, frame_slot_, frame_ctr_, boot_req_, boot_now_, dense_flag_, rescan_req_, rescan_now_,
      taus_, counts_;
  // running max |value| per stream: entry 0 = network input (state of the first
  // layer), entry i+1 = node i's output; the fp16 GEMM scales come from these
  DevBuf amax_;
  // bitmaps written by OR (sparse detections): one arena, zeroed by begin_frame
  DevBuf clear_;
  int n_ext_slots_ = 0;
  int cnt_stride_ = 32;  // ints per stream in counts_  // count slots [0, n_ext_slots_) are uploaded (external nodes), the rest zeroed per frame
  // 8-bit ingest: two staging buffers filled on a copy stream while the other
  // one is being consumed, and three device pointer slots (buffer 0, buffer 1,
  // caller's device pointer) the first detect reads through
  DevBuf frame8_, frame8_slot_;

  cudaStream_t copy_st_ = nullptr;
  cudaEvent_t ev_copied_[2] = {nullptr, nullptr}, ev_consumed_[2] = {nullptr, nullptr};
  int u8_buf_ = 0;
  // host view of the 8-bit state shadow: valid per stream once a full update
  // went through the 8-bit ingest; any fp32 frame invalidates it
  std::vector<uint8_t> s8_valid_, s8_pending_;
  DevBuf delta_stage_[2];
  cudaEvent_t ev_dstaged_[2] = {nullptr, nullptr}, ev_dpushed_[2] = {nullptr, nullptr};
  int delta_buf_ = 0;
  struct DeltaCopy {
    cudaEvent_t ev = nullptr;  // the copy into this host buffer completed
  };
  // apply_output_delta may run on another host thread than the frame / copy
  // calls (a host buffer is handed over by the caller: copy k, then apply k)
  std::mutex delta_mu_;                             // guards delta_host_
  std::map<const void*, DeltaCopy> delta_host_;     // host buffer -> its last copy
  std::atomic<size_t> delta_recent_[4] = {0, 0, 0, 0};  // bytes in use of the last applied deltas
  std::atomic<int> delta_seen_{0};
  size_t delta_dma_last_ = 0;
  DevBuf out_stage_[2];
  cudaEvent_t ev_staged_[2] = {nullptr, nullptr}, ev_drained_[2] = {nullptr, nullptr};
  int out_buf_ = 0;
  void upload_taus(const std::vector<uint8_t>& rescan);
  void run_frame(unsigned flags, unsigned graph_key);
  float* amax_entry(int node) const { return amax_.as<float>() + static_cast<size_t>(node + 1) * S_; }
  int amax_origin(int node) const;  // node whose entry bounds node's output values (pools pass through)
  std::vector<float> ext_amax_;      // host running max of standalone-layer uploads
  int n_slots_ = 0;
  uint32_t host_frame_ = 0;
  unsigned last_flags_ = 0;
  int last_launches_ = 0;
  struct GraphRec {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t begin = nullptr;  // the begin_frame node: its in_ptr is set per launch
    cudaKernelNodeParams begin_params{};
    BeginFrameArgs begin_args{};
  };
  std::map<unsigned, GraphRec> graphs_;
  const void* in_ptr_ = nullptr;      // this frame's input pointer (begin_frame writes it into the slot)
  std::vector<float> host_taus_;      // network thresholds per node (thresholds())
  std::vector<float> stream_taus_;    // [node][S] mirror of the device thresholds
  bool dense_ = false;
  // kernel timing (bench instrumentation)
  template <class F> void timed(const std::string& label, F&& launch, cudaStream_t on = nullptr);
  // Compactions that only read producers' maps (pools, joins, propagate
  // convs) run on a side stream from the moment those maps exist, beside the
  // producer's GEMM; ev_map_[i] = node i's map and list are complete.
  cudaStream_t side_st_ = nullptr;
  std::vector<cudaEvent_t> ev_map_;
  bool side_dc_ = true;
  bool timing_ = false;
  bool dry_ = false;  // kernel_labels(): record labels, launch nothing
  std::vector<std::string> dry_labels_;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending_;
  std::map<std::string, std::pair<double, long long>> times_;
  int timed_frames_ = 0;

};

// Threshold calibration with the replays on the GPU (calib.cpp;
// reference calibration.cpp:95-180).
void select_thresholds(Ctx* ctx, const Topology& topo, const cbg_eval_sequence* seqs, int n_seqs,
                       const cbg_calib_config& cfg, std::vector<float>& taus, std::vector<uint8_t>& hit_cap,
                       std::vector<cbg_calib_trace_point>& trace);
void sweep_threshold_factor(Ctx* ctx, const Topology& topo, const std::vector<float>& base_tau,
                            const std::vector<double>& factors, const cbg_eval_sequence* seqs, int n_seqs, int metric,
                            std::vector<cbg_tradeoff_row>& rows);

}  // namespace cbg
