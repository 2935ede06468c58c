// cbi_gpu.hpp — C++ drop-in for the reference's cbi layer API, running on B200.
//
// Header-only wrapper over the C ABI (include/cbg.h, libcbg.so). It mirrors the
// reference's types and signatures (reference: /root/reference/proj/include/cbi/
// {common,tensor,change,layers,network,io}.hpp) so a caller of
//     cbi::CBNetwork net = cbi::convert_to_cb(cbi::build_network(spec), taus);
//     const cbi::Tensor3& y = net.forward_frame(frame, cfg, &fs);
// switches by changing the namespace to cbg (and linking libcbg.so). Errors are
// the reference's categories (cbg::InvalidInputError / cbg::ConfigError).
//
// Differences a caller may notice:
//  * Device-resident state: the reference's public members prev_output / state
//    are read through prev_output() / state() accessors (synchronising copies).
//  * convert_to_cb also accepts a stream count: one CBNetwork handle may carry
//    S independent camera streams processed by the same launches.
//  * FrameStats rows carry the deterministic fields; wall_ns is 0 (use the
//    CUDA-event timing of the bench instead).
#pragma once

#include <algorithm>
#include <cstdint>
#include <ostream>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../cbg.h"

namespace cbg {

// ---- errors (common.hpp:11-21) ----------------------------------------------------
class InvalidInputError : public std::runtime_error {
 public:
  explicit InvalidInputError(const std::string& m) : std::runtime_error(m) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int status) {
  if (status == CBG_OK) return;
  const std::string msg = cbg_last_error();
  if (status == CBG_ERR_INVALID_INPUT) throw InvalidInputError(msg);
  if (status == CBG_ERR_CONFIG) throw ConfigError(msg);
  throw DeviceError(msg);
}

// ---- tensors (tensor.hpp:13-116, change.hpp:11-25) -----------------------------------
struct Tensor3 {
  int channels = 0, height = 0, width = 0;
  std::vector<float> data;
  Tensor3() = default;
  Tensor3(int c, int h, int w) : channels(c), height(h), width(w), data(static_cast<size_t>(c) * h * w, 0.0f) {}
  float& at(int c, int j, int i) { return data[(static_cast<size_t>(c) * height + j) * width + i]; }
  float at(int c, int j, int i) const { return data[(static_cast<size_t>(c) * height + j) * width + i]; }
  size_t size() const { return data.size(); }
  bool same_shape(const Tensor3& o) const { return channels == o.channels && height == o.height && width == o.width; }
};

struct PixelIndex {
  int row = 0, col = 0;
  bool operator==(const PixelIndex& o) const { return row == o.row && col == o.col; }
};
using IndexList = std::vector<PixelIndex>;

struct ChangeMap {
  int height = 0, width = 0;
  std::vector<uint8_t> bits;
  ChangeMap() = default;
  ChangeMap(int h, int w) : height(h), width(w), bits(static_cast<size_t>(h) * w, 0) {}
  uint8_t at(int j, int i) const { return bits[static_cast<size_t>(j) * width + i]; }
  int64_t count() const {
    int64_t n = 0;
    for (uint8_t b : bits) n += b != 0;
    return n;
  }
  bool operator==(const ChangeMap& o) const { return height == o.height && width == o.width && bits == o.bits; }
};

struct ConvSpec {
  int in_channels = 0, out_channels = 0, kernel_h = 0, kernel_w = 0, stride = 1, padding = 0;
  int out_h = 0, out_w = 0;
  std::vector<float> weights, bias;
  size_t weight_count() const {
    return static_cast<size_t>(out_channels) * in_channels * kernel_h * kernel_w;
  }
  cbg_conv_spec c() const {
    return cbg_conv_spec{in_channels, out_channels, kernel_h, kernel_w, stride, padding, out_h, out_w,
                         weights.data(), bias.data()};
  }
};

enum class DetectionPolicy { Detect = CBG_POLICY_DETECT, Propagate = CBG_POLICY_PROPAGATE, Reuse1x1 = CBG_POLICY_REUSE1X1 };
enum class DetectMode { FeedForward = CBG_MODE_FEEDFORWARD, ClosedLoop = CBG_MODE_CLOSEDLOOP };
enum class LayerKind { Conv = CBG_LAYER_CONV, Act = CBG_LAYER_ACT, Pool = CBG_LAYER_POOL, Add = CBG_LAYER_ADD, Concat = CBG_LAYER_CONCAT,
                       Upsample = CBG_LAYER_UPSAMPLE /* extension: not in the reference */ };

// ---- device context -----------------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) {
    cbg_ctx h = nullptr;
    check(cbg_ctx_create(device, &h));
    h_.reset(h, cbg_ctx_destroy);
  }
  static std::shared_ptr<Context> default_context() {
    static std::shared_ptr<Context> ctx = std::make_shared<Context>(0);
    return ctx;
  }
  cbg_ctx handle() const { return h_.get(); }
  void synchronize() const { check(cbg_ctx_sync(h_.get())); }

 private:
  std::shared_ptr<cbg_ctx_s> h_;
};

// ---- layers (layers.hpp:8-91) -------------------------------------------------------------
struct UpstreamChange {
  const ChangeMap* map = nullptr;
  const IndexList* indexes = nullptr;
};

struct ConvForwardOptions {
  bool force_full_update = false;
  bool record_worst_case = false;
  bool estimate_fg = false;  // analytics, not part of the hot path: ignored
};

struct ConvForwardResult {
  ChangeMap out_map;
  IndexList indexes;
  int64_t eff_ops = 0;
  ChangeMap worst_case_map;
  int64_t propagated_px = -1;
  int64_t fg_sp_ops = -1;
  int64_t fg_fm_ops = -1;
};

struct PoolForwardResult {
  ChangeMap out_map;
  IndexList indexes;
};

namespace detail {
inline std::vector<int32_t> rowcol(const IndexList* idx) {
  std::vector<int32_t> v;
  if (!idx) return v;
  v.reserve(idx->size() * 2);
  for (const PixelIndex& p : *idx) {
    v.push_back(p.row);
    v.push_back(p.col);
  }
  return v;
}
inline IndexList to_indexes(const std::vector<int32_t>& rc, int64_t n) {
  IndexList l(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) l[k] = {rc[2 * k], rc[2 * k + 1]};
  return l;
}
}  // namespace detail

class CBConvLayer {
 public:
  CBConvLayer(ConvSpec s, float tau, DetectionPolicy policy, bool fuse_relu, DetectMode mode, int in_height,
              int in_width, std::shared_ptr<Context> ctx = Context::default_context())
      : spec(std::move(s)), tau_(tau), policy(policy), fuse_relu(fuse_relu), mode(mode), in_h(in_height),
        in_w(in_width), ctx_(std::move(ctx)) {
    const cbg_conv_spec cs = spec.c();
    cbg_conv h = nullptr;
    check(cbg_conv_create(ctx_->handle(), &cs, tau, static_cast<int>(policy), fuse_relu ? 1 : 0,
                          static_cast<int>(mode), in_h, in_w, &h));
    h_.reset(h, cbg_conv_destroy);
    check(cbg_conv_out_dims(h, &out_h, &out_w));
  }

  // CBConvLayer::forward, layers.cpp:55-131
  ConvForwardResult forward(const Tensor3& x, const UpstreamChange& up, const ConvForwardOptions& opt = {}) {
    if (x.channels != spec.in_channels || x.height != in_h || x.width != in_w)
      throw InvalidInputError("CBConvLayer: input shape mismatch");
    const std::vector<int32_t> rc = detail::rowcol(up.indexes);
    const unsigned flags = (opt.force_full_update ? CBG_FWD_FORCE_FULL : 0u) |
                           (opt.record_worst_case ? CBG_FWD_RECORD_WORST_CASE : 0u);
    ConvForwardResult r;
    check(cbg_conv_forward(h_.get(), x.data.data(), up.map ? up.map->bits.data() : nullptr,
                           up.indexes ? rc.data() : nullptr, up.indexes ? static_cast<int64_t>(up.indexes->size()) : 0,
                           flags, &r.eff_ops));
    r.out_map = ChangeMap(out_h, out_w);
    std::vector<int32_t> out_rc(static_cast<size_t>(out_h) * out_w * 2);
    int64_t n = 0;
    check(cbg_conv_read_changes(h_.get(), r.out_map.bits.data(), out_rc.data(), &n));
    r.indexes = detail::to_indexes(out_rc, n);
    if (opt.record_worst_case) {
      r.worst_case_map = ChangeMap(out_h, out_w);
      check(cbg_conv_read_worst_case(h_.get(), r.worst_case_map.bits.data(), &r.propagated_px));
    }
    return r;
  }

  Tensor3 prev_output() const {
    Tensor3 t(spec.out_channels, out_h, out_w);
    check(cbg_conv_read_output(h_.get(), t.data.data()));
    return t;
  }
  Tensor3 state() const {
    Tensor3 t(spec.in_channels, in_h, in_w);
    check(cbg_conv_read_state(h_.get(), t.data.data()));
    return t;
  }
  float tau() const { return tau_; }
  void set_tau(float t) {
    check(cbg_conv_set_tau(h_.get(), t));
    tau_ = t;
  }
  int64_t ops_per_pixel() const {
    return 2ll * spec.out_channels * spec.in_channels * spec.kernel_h * spec.kernel_w;
  }
  int64_t dense_ops() const { return ops_per_pixel() * out_h * out_w; }

  ConvSpec spec;

 private:
  float tau_;

 public:
  DetectionPolicy policy;
  bool fuse_relu;
  DetectMode mode;
  int in_h = 0, in_w = 0, out_h = 0, out_w = 0;

 private:
  std::shared_ptr<Context> ctx_;
  std::shared_ptr<cbg_conv_s> h_;
};

class CBPoolLayer {
 public:
  CBPoolLayer(int size_, int stride_, int channels_, int in_height, int in_width, int out_height, int out_width,
              std::shared_ptr<Context> ctx = Context::default_context())
      : size(size_), stride(stride_), channels(channels_), in_h(in_height), in_w(in_width), out_h(out_height),
        out_w(out_width), ctx_(std::move(ctx)) {
    cbg_pool h = nullptr;
    check(cbg_pool_create(ctx_->handle(), size, stride, channels, in_h, in_w, out_h, out_w, &h));
    h_.reset(h, cbg_pool_destroy);
  }

  // CBPoolLayer::forward, layers.cpp:148-179
  PoolForwardResult forward(const Tensor3& x, const UpstreamChange& up, bool force_full_update = false) {
    if (x.channels != channels || x.height != in_h || x.width != in_w)
      throw InvalidInputError("CBPoolLayer: input shape mismatch");
    const std::vector<int32_t> rc = detail::rowcol(up.indexes);
    check(cbg_pool_forward(h_.get(), x.data.data(), up.map ? up.map->bits.data() : nullptr,
                           up.indexes ? rc.data() : nullptr, up.indexes ? static_cast<int64_t>(up.indexes->size()) : 0,
                           force_full_update ? 1 : 0));
    PoolForwardResult r;
    r.out_map = ChangeMap(out_h, out_w);
    std::vector<int32_t> out_rc(static_cast<size_t>(out_h) * out_w * 2);
    int64_t n = 0;
    check(cbg_pool_read_changes(h_.get(), r.out_map.bits.data(), out_rc.data(), &n));
    r.indexes = detail::to_indexes(out_rc, n);
    return r;
  }
  Tensor3 prev_output() const {
    Tensor3 t(channels, out_h, out_w);
    check(cbg_pool_read_output(h_.get(), t.data.data()));
    return t;
  }

  int size, stride, channels, in_h, in_w, out_h, out_w;

 private:
  std::shared_ptr<Context> ctx_;
  std::shared_ptr<cbg_pool_s> h_;
};

// ---- network (network.hpp:10-195) ------------------------------------------------------------
struct LayerDesc {
  LayerKind kind = LayerKind::Conv;
  std::string name;
  std::vector<std::string> from;
  ConvSpec conv;
  bool fuse_relu = false;
  int pool_size = 0, pool_stride = 0, pool_out_h = 0, pool_out_w = 0;
  float act_slope = 0.0f;  // extension: leaky ReLU slope of an Act row / fused activation (0 = ReLU)
  int upsample = 0;        // extension: Upsample rows' factor
};

struct NetworkSpec {
  int in_channels = 0, in_height = 0, in_width = 0;
  std::vector<LayerDesc> layers;
};

// The reference's DenseNetwork is its CPU oracle; here it only carries the spec
// so convert_to_cb(build_network(spec), taus) keeps compiling.
class DenseNetwork {
 public:
  explicit DenseNetwork(NetworkSpec s) : spec_(std::move(s)) {}
  const NetworkSpec& spec() const { return spec_; }

 private:
  NetworkSpec spec_;
};
inline DenseNetwork build_network(NetworkSpec spec) { return DenseNetwork(std::move(spec)); }

struct StatsConfig {
  bool record_worst_case = false;
  bool record_maps = false;
  bool estimate_fg = false;
  bool timing = true;
};

struct LayerFrameStats {
  std::string layer;
  int64_t changed_px = 0, total_px = 0;
  double change_frac = 0.0;
  int64_t eff_ops = 0, wall_ns = 0, propagated_px = -1, fg_sp_ops = -1, fg_fm_ops = -1;
  ChangeMap map, worst_case_map;
};

struct FrameStats {
  int frame = 0;
  bool has_loss = false;
  double loss = 0.0;
  std::vector<LayerFrameStats> layers;
};

namespace detail {
// Keeps the C description structs (and the strings they point to) alive.
struct CSpec {
  std::vector<cbg_layer_desc> layers;
  std::vector<std::vector<const char*>> from;
  cbg_network_spec spec{};
  explicit CSpec(const NetworkSpec& s) {
    layers.resize(s.layers.size());
    from.resize(s.layers.size());
    for (size_t i = 0; i < s.layers.size(); ++i) {
      const LayerDesc& d = s.layers[i];
      for (const std::string& f : d.from) from[i].push_back(f.c_str());
      cbg_layer_desc& c = layers[i];
      c.kind = static_cast<int>(d.kind);
      c.name = d.name.c_str();
      c.n_from = static_cast<int>(d.from.size());
      c.from = from[i].data();
      c.conv = d.conv.c();
      c.fuse_relu = d.fuse_relu ? 1 : 0;
      c.pool_size = d.pool_size;
      c.pool_stride = d.pool_stride;
      c.pool_out_h = d.pool_out_h;
      c.pool_out_w = d.pool_out_w;
      c.act_slope = d.act_slope;
      c.upsample = d.upsample;
    }
    spec = cbg_network_spec{s.in_channels, s.in_height, s.in_width, static_cast<int>(layers.size()), layers.data()};
  }
};
}  // namespace detail

class CBNetwork {
 public:
  CBNetwork() = default;

  int stream_count() const { return streams_; }
  int node_count() const { return static_cast<int>(info_.size()); }
  const cbg_node_info& node(int i) const { return info_[i]; }
  int conv_layer_count() const {
    int n = 0;
    for (const cbg_node_info& i : info_) n += i.kind == CBG_LAYER_CONV;
    return n;
  }

  std::vector<float> thresholds() const {
    std::vector<float> t(static_cast<size_t>(conv_layer_count()));
    check(cbg_net_thresholds(h_.get(), t.data(), static_cast<int>(t.size())));
    return t;
  }
  void set_thresholds(const std::vector<float>& taus) {
    check(cbg_net_set_thresholds(h_.get(), taus.data(), static_cast<int>(taus.size())));
  }
  // network.cpp:274-290 (stream = -1: all streams)
  void reset(int stream = -1) { check(cbg_net_reset(h_.get(), stream)); }

  // forward_frame, network.cpp:309-414 (single-stream networks)
  const Tensor3& forward_frame(const Tensor3& frame, const StatsConfig& cfg = {}, FrameStats* fs = nullptr) {
    const cbg_node_info& n0 = info_.front();
    if (frame.channels != n0.in_channels || frame.height != n0.in_height || frame.width != n0.in_width)
      throw InvalidInputError("forward_frame: frame resolution mismatch");
    if (streams_ != 1) throw InvalidInputError("forward_frame: use forward_frames for multi-stream networks");
    check(cbg_net_forward(h_.get(), frame.data.data(), cfg.record_worst_case ? CBG_FWD_RECORD_WORST_CASE : 0u));
    ++frame_no_;
    if (fs) fill_stats(0, cfg, fs);
    out_ = output(0);
    return out_;
  }
  // One frame per stream, all streams in one step (frames: S x C x H x W contiguous).
  void forward_frames(const float* frames, bool frames_on_device = false) {
    check(cbg_net_forward(h_.get(), frames, frames_on_device ? CBG_FWD_INPUT_ON_DEVICE : 0u));
    ++frame_no_;
  }

  Tensor3 output(int stream = 0) const { return node_output(node_count() - 1, stream); }
  Tensor3 node_output(int node, int stream = 0) const {
    const cbg_node_info& i = info_[node];
    Tensor3 t(i.out_channels, i.out_height, i.out_width);
    check(cbg_net_read_output(h_.get(), node, stream, t.data.data()));
    return t;
  }
  Tensor3 node_state(int node, int stream = 0) const {
    const cbg_node_info& i = info_[node];
    Tensor3 t(i.in_channels, i.in_height, i.in_width);
    check(cbg_net_read_state(h_.get(), node, stream, t.data.data()));
    return t;
  }
  std::pair<ChangeMap, IndexList> node_changes(int node, int stream = 0) const {
    const cbg_node_info& i = info_[node];
    ChangeMap m(i.out_height, i.out_width);
    std::vector<int32_t> rc(static_cast<size_t>(i.out_height) * i.out_width * 2);
    int64_t n = 0;
    check(cbg_net_read_changes(h_.get(), node, stream, m.bits.data(), rc.data(), &n));
    return {m, detail::to_indexes(rc, n)};
  }

  // One stream's thresholds (the others keep theirs).
  void set_stream_thresholds(int stream, const std::vector<float>& taus) {
    check(cbg_net_set_stream_thresholds(h_.get(), stream, taus.data(), static_cast<int>(taus.size())));
  }
  cbg_net handle() const { return h_.get(); }

  CBNetwork clone() const {
    CBNetwork c;
    cbg_net h = nullptr;
    check(cbg_net_clone(h_.get(), &h));
    c.h_.reset(h, cbg_net_destroy);
    c.ctx_ = ctx_;
    c.info_ = info_;
    c.streams_ = streams_;
    c.frame_no_ = frame_no_;
    return c;
  }

  friend CBNetwork convert_to_cb(const DenseNetwork& net, const std::vector<float>& taus,
                                 const std::vector<DetectionPolicy>* policies, DetectMode mode, int n_streams,
                                 std::shared_ptr<Context> ctx);

 private:
  void fill_stats(int stream, const StatsConfig& cfg, FrameStats* fs) {
    std::vector<cbg_layer_stats> st(info_.size());
    check(cbg_net_read_stats(h_.get(), stream, st.data(), static_cast<int>(st.size())));
    fs->frame = frame_no_;
    fs->layers.clear();
    for (size_t i = 0; i < st.size(); ++i) {
      LayerFrameStats row;
      row.layer = info_[i].name;
      row.changed_px = st[i].changed_px;
      row.total_px = st[i].total_px;
      row.change_frac = st[i].total_px ? static_cast<double>(st[i].changed_px) / st[i].total_px : 0.0;
      row.eff_ops = st[i].eff_ops;
      row.propagated_px = st[i].propagated_px;
      if (cfg.record_maps) row.map = node_changes(static_cast<int>(i), stream).first;
      fs->layers.push_back(std::move(row));
    }
  }

  std::shared_ptr<Context> ctx_;
  std::shared_ptr<cbg_net_s> h_;
  std::vector<cbg_node_info> info_;
  int streams_ = 1;
  int frame_no_ = 0;
  Tensor3 out_;
};

// convert_to_cb, network.cpp:416-503 (+ stream count for multi-stream sets)
inline CBNetwork convert_to_cb(const DenseNetwork& net, const std::vector<float>& taus,
                               const std::vector<DetectionPolicy>* policies = nullptr,
                               DetectMode mode = DetectMode::ClosedLoop, int n_streams = 1,
                               std::shared_ptr<Context> ctx = Context::default_context()) {
  detail::CSpec cs(net.spec());
  std::vector<int> pol;
  if (policies)
    for (DetectionPolicy p : *policies) pol.push_back(static_cast<int>(p));
  cbg_net h = nullptr;
  check(cbg_net_create(ctx->handle(), &cs.spec, taus.data(), static_cast<int>(taus.size()),
                       policies ? pol.data() : nullptr, static_cast<int>(mode), n_streams, &h));
  CBNetwork cb;
  cb.h_.reset(h, cbg_net_destroy);
  cb.ctx_ = std::move(ctx);
  cb.streams_ = n_streams;
  int n = 0;
  check(cbg_net_node_count(h, &n));
  cb.info_.resize(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) check(cbg_net_node_info(h, i, &cb.info_[i]));
  return cb;
}

// ---- calibration (calibration.hpp:16-84), replays on the GPU --------------------
enum class LossMetric { Mse, PixelAccuracyDelta };

// ---- sequences and stats CSV (network.hpp:119-126,183-195; io.cpp:660-672) --------
struct RunStats {
  std::vector<FrameStats> frames;
  std::int64_t total_eff_ops(int first_frame = 1) const {
    std::int64_t n = 0;
    for (const FrameStats& f : frames)
      if (f.frame >= first_frame)
        for (const LayerFrameStats& l : f.layers) n += l.eff_ops;
    return n;
  }
};
struct SequenceResult {
  std::vector<Tensor3> outputs;
  RunStats stats;
};

namespace detail {
inline int argmax_channel(const Tensor3& t, int j, int i) {  // calibration.cpp:11-22
  int best = 0;
  float best_v = t.at(0, j, i);
  for (int c = 1; c < t.channels; ++c)
    if (t.at(c, j, i) > best_v) best_v = t.at(c, j, i), best = c;
  return best;
}
// loss_value, calibration.cpp:26-53
inline double loss_value(LossMetric metric, const Tensor3& pred, const Tensor3& ref) {
  if (metric == LossMetric::Mse) {
    if (pred.channels != ref.channels || pred.height != ref.height || pred.width != ref.width)
      throw InvalidInputError("mse: shapes differ");
    double acc = 0.0;
    for (size_t i = 0; i < pred.data.size(); ++i) {
      const double d = static_cast<double>(pred.data[i]) - ref.data[i];
      acc += d * d;
    }
    return acc / static_cast<double>(pred.data.size());
  }
  if (pred.height != ref.height || pred.width != ref.width) throw InvalidInputError("pixel_accuracy: spatial dims differ");
  if (ref.channels != 1 && ref.channels != pred.channels)
    throw InvalidInputError("pixel_accuracy: reference channels must be 1 (labels) or match");
  std::int64_t hits = 0;
  for (int j = 0; j < pred.height; ++j)
    for (int i = 0; i < pred.width; ++i)
      hits += argmax_channel(pred, j, i) ==
              (ref.channels == 1 ? static_cast<int>(ref.at(0, j, i)) : argmax_channel(ref, j, i));
  return 1.0 - static_cast<double>(hits) / (static_cast<std::int64_t>(pred.height) * pred.width);
}
}  // namespace detail

// forward_sequence, network.cpp:505-525
inline SequenceResult forward_sequence(CBNetwork& net, const std::vector<Tensor3>& frames,
                                       const std::vector<Tensor3>* reference = nullptr,
                                       LossMetric metric = LossMetric::Mse, const StatsConfig& cfg = {}) {
  if (reference && reference->size() != frames.size())
    throw InvalidInputError("forward_sequence: reference count != frame count");
  SequenceResult result;
  for (size_t t = 0; t < frames.size(); ++t) {
    FrameStats fs;
    const Tensor3& out = net.forward_frame(frames[t], cfg, &fs);
    fs.frame = static_cast<int>(t) + 1;
    if (reference) {
      fs.loss = detail::loss_value(metric, out, (*reference)[t]);
      fs.has_loss = true;
    }
    result.outputs.push_back(out);
    result.stats.frames.push_back(std::move(fs));
  }
  return result;
}

// write_stats_csv, io.cpp:660-672 (same columns and number formats)
inline void write_stats_csv(std::ostream& os, const RunStats& run) {
  os << "frame,layer,changed_px,change_frac,eff_ops,wall_ns,loss\n";
  char frac[32], loss[48];
  for (const FrameStats& f : run.frames)
    for (const LayerFrameStats& l : f.layers) {
      std::snprintf(frac, sizeof frac, "%.6f", l.change_frac);
      os << f.frame << "," << l.layer << "," << l.changed_px << "," << frac << "," << l.eff_ops << "," << l.wall_ns
         << ",";
      if (f.has_loss) {
        std::snprintf(loss, sizeof loss, "%.9g", f.loss);
        os << loss;
      }
      os << "\n";
    }
}
enum class LossAggregation { Mean, Worst };

struct EvalSequence {
  std::vector<Tensor3> frames;
  std::vector<Tensor3> reference;
};

struct CalibConfig {
  double initial_tau = 0.01;
  double growth_factor = 1.1;
  double per_layer_budget = 0.0;
  std::vector<double> budget_overrides;
  LossMetric metric = LossMetric::Mse;
  LossAggregation aggregation = LossAggregation::Mean;
  int max_steps = 64;
};

struct CalibTracePoint {
  int layer = 0;
  double tau = 0.0;
  double loss = 0.0;
};

struct CalibResult {
  std::vector<float> taus;
  std::vector<bool> hit_cap;
  std::vector<CalibTracePoint> trace;
};

struct TradeoffRow {
  double factor = 0.0;
  double loss = 0.0;
  std::int64_t total_eff_ops = 0;
  std::int64_t wall_ns = 0;
};

namespace detail {
// Flattened host copies of the sequences for the C ABI.
struct CSequences {
  std::vector<std::vector<float>> f, r;
  std::vector<cbg_eval_sequence> v;
  explicit CSequences(const std::vector<EvalSequence>& seqs) {
    for (const EvalSequence& q : seqs) {
      if (q.frames.empty() || q.reference.size() != q.frames.size())
        throw InvalidInputError("calibration sequence needs frames and per-frame references");
      f.emplace_back();
      r.emplace_back();
      for (const Tensor3& t : q.frames) f.back().insert(f.back().end(), t.data.begin(), t.data.end());
      for (const Tensor3& t : q.reference) r.back().insert(r.back().end(), t.data.begin(), t.data.end());
      v.push_back({static_cast<int>(q.frames.size()), f.back().data(), r.back().data(), q.reference[0].channels});
    }
  }
};
}  // namespace detail

// select_thresholds, calibration.cpp:95-141
inline CalibResult select_thresholds(const CBNetwork& net, const std::vector<EvalSequence>& sequences,
                                     const CalibConfig& cfg) {
  detail::CSequences cs(sequences);
  cbg_calib_config c{cfg.initial_tau, cfg.growth_factor, cfg.per_layer_budget,
                     cfg.budget_overrides.empty() ? nullptr : cfg.budget_overrides.data(),
                     static_cast<int>(cfg.budget_overrides.size()), static_cast<int>(cfg.metric),
                     static_cast<int>(cfg.aggregation), cfg.max_steps};
  const int n_conv = net.conv_layer_count();
  std::vector<float> taus(static_cast<size_t>(n_conv));
  std::vector<uint8_t> cap(static_cast<size_t>(n_conv));
  std::vector<cbg_calib_trace_point> tr(static_cast<size_t>(std::max(1, n_conv * std::max(1, cfg.max_steps))));
  int n = 0;
  check(cbg_select_thresholds(net.handle(), cs.v.data(), static_cast<int>(cs.v.size()), &c, taus.data(), cap.data(),
                              tr.data(), static_cast<int>(tr.size()), &n));
  CalibResult res;
  res.taus = taus;
  for (uint8_t b : cap) res.hit_cap.push_back(b != 0);
  for (int i = 0; i < n && i < static_cast<int>(tr.size()); ++i) res.trace.push_back({tr[i].layer, tr[i].tau, tr[i].loss});
  return res;
}

// sweep_threshold_factor, calibration.cpp:143-180
inline std::vector<TradeoffRow> sweep_threshold_factor(const CBNetwork& net, const std::vector<float>& base_tau,
                                                       const std::vector<double>& factors,
                                                       const std::vector<EvalSequence>& sequences,
                                                       LossMetric metric = LossMetric::Mse) {
  detail::CSequences cs(sequences);
  std::vector<cbg_tradeoff_row> rows(factors.size());
  check(cbg_sweep_threshold_factor(net.handle(), base_tau.data(), static_cast<int>(base_tau.size()), factors.data(),
                                   static_cast<int>(factors.size()), cs.v.data(), static_cast<int>(cs.v.size()),
                                   static_cast<int>(metric), rows.data()));
  std::vector<TradeoffRow> out;
  for (const cbg_tradeoff_row& r : rows) out.push_back({r.factor, r.loss, r.total_eff_ops, r.wall_ns});
  return out;
}

}  // namespace cbg
