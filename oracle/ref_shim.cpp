// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the product.
//
// A C entry-point shim over the UNMODIFIED reference library (cbi, compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/). It lets the
// pytest parity suite, golden-vector generator and bench.py's cpu_baseline leg
// drive the reference with exactly the inputs our GPU path sees. Only tests/,
// __graft_entry__.smoke() and bench.py's CPU leg may load it.
//
// Entry points mirror the reference API 1:1 (cited per function) and reuse the
// cbg_* description structs of include/cbg.h so both sides are fed the same data.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "cbg.h"
#include <algorithm>
#include <sstream>

#include "cbi/calibration.hpp"
#include "cbi/change.hpp"
#include "cbi/dense.hpp"
#include "cbi/io.hpp"
#include "cbi/layers.hpp"
#include "cbi/network.hpp"

using namespace cbi;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return CBG_OK;
  } catch (const InvalidInputError& e) {
    g_err = e.what();
    return CBG_ERR_INVALID_INPUT;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return CBG_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CBG_ERR_CUDA;
  }
}

ConvSpec to_spec(const cbg_conv_spec& c) {
  ConvSpec s;
  s.in_channels = c.in_channels;
  s.out_channels = c.out_channels;
  s.kernel_h = c.kernel_h;
  s.kernel_w = c.kernel_w;
  s.stride = c.stride;
  s.padding = c.padding;
  s.out_h = c.out_h;
  s.out_w = c.out_w;
  const std::size_t nw = static_cast<std::size_t>(c.out_channels > 0 ? c.out_channels : 0) *
                         (c.in_channels > 0 ? c.in_channels : 0) *
                         (c.kernel_h > 0 ? c.kernel_h : 0) * (c.kernel_w > 0 ? c.kernel_w : 0);
  if (c.weights) s.weights.assign(c.weights, c.weights + nw);
  else s.weights.assign(nw, 0.0f);
  if (c.bias) s.bias.assign(c.bias, c.bias + (c.out_channels > 0 ? c.out_channels : 0));
  else s.bias.assign(c.out_channels > 0 ? c.out_channels : 0, 0.0f);
  return s;
}

NetworkSpec to_network(const cbg_network_spec& n) {
  NetworkSpec spec;
  spec.in_channels = n.in_channels;
  spec.in_height = n.in_height;
  spec.in_width = n.in_width;
  for (int i = 0; i < n.n_layers; ++i) {
    const cbg_layer_desc& d = n.layers[i];
    if (d.kind == CBG_LAYER_UPSAMPLE || d.act_slope != 0.0f)
      throw ConfigError("the reference has no upsample layer and no leaky ReLU (network.hpp:10)");
    LayerDesc l;
    l.kind = static_cast<LayerKind>(d.kind);
    l.name = d.name ? d.name : "";
    for (int k = 0; k < d.n_from; ++k) l.from.push_back(d.from[k]);
    if (d.kind == CBG_LAYER_CONV) l.conv = to_spec(d.conv);
    l.fuse_relu = d.fuse_relu != 0;
    l.pool_size = d.pool_size;
    l.pool_stride = d.pool_stride;
    l.pool_out_h = d.pool_out_h;
    l.pool_out_w = d.pool_out_w;
    spec.layers.push_back(std::move(l));
  }
  return spec;
}

Tensor3 to_tensor(const float* p, int c, int h, int w) {
  Tensor3 t(c, h, w);
  std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
  return t;
}

void put_tensor(const Tensor3& t, float* out) {
  std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}

ChangeMap to_map(const uint8_t* bits, int h, int w) {
  ChangeMap m(h, w);
  for (std::size_t i = 0; i < m.bits.size(); ++i) m.bits[i] = bits[i] ? 1 : 0;
  return m;
}

IndexList to_idx(const int32_t* rc, int64_t n) {
  IndexList l;
  for (int64_t k = 0; k < n; ++k) l.push_back({rc[2 * k], rc[2 * k + 1]});
  return l;
}

void put_idx(const IndexList& l, int32_t* rc) {
  for (std::size_t k = 0; k < l.size(); ++k) {
    rc[2 * k] = l[k].row;
    rc[2 * k + 1] = l[k].col;
  }
}

struct RefNet {
  std::unique_ptr<DenseNetwork> dense;
  CBNetwork cb;
  FrameStats last;
  bool record_maps = true;
};

struct RefConv {
  CBConvLayer layer;
  ConvForwardResult last;
};

struct RefPool {
  CBPoolLayer layer;
  PoolForwardResult last;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// gen_synthetic, io.cpp:499-552
int ref_gen_synthetic(const cbg_synthetic_config* c, float* frames_out, int32_t* corners_out) {
  return guard([&] {
    SyntheticConfig cfg;
    cfg.height = c->height;
    cfg.width = c->width;
    cfg.channels = c->channels;
    cfg.n_frames = c->n_frames;
    cfg.n_objects = c->n_objects;
    cfg.object_size = c->object_size;
    cfg.velocity_y = c->velocity_y;
    cfg.velocity_x = c->velocity_x;
    cfg.noise_std = c->noise_std;
    cfg.seed = c->seed;
    std::vector<std::vector<PixelIndex>> corners;
    std::vector<Tensor3> fr = gen_synthetic(cfg, corners_out ? &corners : nullptr);
    std::size_t off = 0;
    for (const Tensor3& t : fr) {
      std::memcpy(frames_out + off, t.data.data(), t.data.size() * sizeof(float));
      off += t.data.size();
    }
    if (corners_out) {
      std::size_t k = 0;
      for (const auto& f : corners)
        for (const PixelIndex& p : f) {
          corners_out[k++] = p.row;
          corners_out[k++] = p.col;
        }
    }
  });
}

// fill_random_weights, io.cpp:554-566
int ref_fill_random_weights(const cbg_network_spec* n, uint32_t seed, float* const* w,
                            float* const* b) {
  return guard([&] {
    NetworkSpec spec = to_network(*n);
    fill_random_weights(spec, seed);
    int k = 0;
    for (const LayerDesc& d : spec.layers) {
      if (d.kind != LayerKind::Conv) continue;
      std::memcpy(w[k], d.conv.weights.data(), d.conv.weights.size() * sizeof(float));
      std::memcpy(b[k], d.conv.bias.data(), d.conv.bias.size() * sizeof(float));
      ++k;
    }
  });
}

// ---- primitives --------------------------------------------------------------
// detect_changes, change.cpp:20-43. state is updated in place.
int ref_detect_changes(const float* x, float* state, int c, int h, int w, float tau, int mode,
                       uint8_t* map_out) {
  return guard([&] {
    InputState st{to_tensor(state, c, h, w)};
    ChangeMap m = detect_changes(to_tensor(x, c, h, w), st, tau, static_cast<DetectMode>(mode));
    put_tensor(st.state, state);
    std::memcpy(map_out, m.bits.data(), m.bits.size());
  });
}

// dilate_window, change.cpp:45-61
int ref_dilate_window(const uint8_t* m, int h, int w, int kh, int kw, int stride, int pad,
                      int oh, int ow, uint8_t* out) {
  return guard([&] {
    ChangeMap d = dilate_window(to_map(m, h, w), kh, kw, stride, pad, oh, ow);
    std::memcpy(out, d.bits.data(), d.bits.size());
  });
}

// propagate_changes, change.cpp:69-75
int ref_propagate_changes(const uint8_t* m, int h, int w, const cbg_conv_spec* s, uint8_t* out,
                          int* oh, int* ow) {
  return guard([&] {
    ChangeMap d = propagate_changes(to_map(m, h, w), to_spec(*s));
    *oh = d.height;
    *ow = d.width;
    if (out) std::memcpy(out, d.bits.data(), d.bits.size());
  });
}

// extract_indexes, change.cpp:77-84
int ref_extract_indexes(const uint8_t* m, int h, int w, int32_t* rc, int64_t* n) {
  return guard([&] {
    IndexList l = extract_indexes(to_map(m, h, w));
    *n = static_cast<int64_t>(l.size());
    if (rc) put_idx(l, rc);
  });
}

// conv2d_dense, dense.cpp:8-42
int ref_conv2d_dense(const float* x, int c, int h, int w, const cbg_conv_spec* s, float* y) {
  return guard([&] { put_tensor(conv2d_dense(to_tensor(x, c, h, w), to_spec(*s)), y); });
}

// im2col, dense.cpp:44-83 (column-major [rows][cols] -> written as data order)
int ref_im2col(const float* x, int c, int h, int w, const cbg_conv_spec* s, const int32_t* rc,
               int64_t n, float* cols_out) {
  return guard([&] {
    IndexList sel = to_idx(rc, n);
    ColumnMatrix m = im2col(to_tensor(x, c, h, w), to_spec(*s), rc ? &sel : nullptr);
    std::memcpy(cols_out, m.data.data(), m.data.size() * sizeof(float));
  });
}

// gemm(make_kernel_matrix(spec), X), dense.cpp:85-112 / tensor.cpp:45-56
int ref_gemm(const cbg_conv_spec* s, const float* cols, int64_t n, float* y) {
  return guard([&] {
    ConvSpec spec = to_spec(*s);
    ColumnMatrix x;
    x.rows = spec.in_channels * spec.kernel_h * spec.kernel_w;
    x.cols = static_cast<int>(n);
    x.data.assign(cols, cols + static_cast<std::size_t>(x.rows) * x.cols);
    Matrix r = gemm(make_kernel_matrix(spec), x);
    std::memcpy(y, r.data.data(), r.data.size() * sizeof(float));
  });
}

// maxpool_to, dense.cpp:125-145
int ref_maxpool_to(const float* x, int c, int h, int w, int size, int stride, int oh, int ow,
                   float* y) {
  return guard([&] { put_tensor(maxpool_to(to_tensor(x, c, h, w), size, stride, oh, ow), y); });
}

// ---- layers --------------------------------------------------------------------
// CBConvLayer ctor, layers.cpp:33-53
int ref_conv_create(const cbg_conv_spec* s, float tau, int policy, int relu, int mode, int in_h,
                    int in_w, void** out) {
  return guard([&] {
    auto* r = new RefConv{CBConvLayer(to_spec(*s), tau, static_cast<DetectionPolicy>(policy),
                                      relu != 0, static_cast<DetectMode>(mode), in_h, in_w),
                          {}};
    *out = r;
  });
}
void ref_conv_destroy(void* h) { delete static_cast<RefConv*>(h); }

// CBConvLayer::forward, layers.cpp:55-131
int ref_conv_forward(void* h, const float* x, const uint8_t* up_map, const int32_t* up_rc,
                     int64_t up_n, unsigned flags, int64_t* eff_ops) {
  auto* r = static_cast<RefConv*>(h);
  return guard([&] {
    CBConvLayer& L = r->layer;
    ChangeMap m;
    IndexList idx;
    UpstreamChange up;
    if (up_map) {
      m = to_map(up_map, L.in_h, L.in_w);
      up.map = &m;
    }
    if (up_rc) {
      idx = to_idx(up_rc, up_n);
      up.indexes = &idx;
    }
    ConvForwardOptions opt;
    opt.force_full_update = (flags & CBG_FWD_FORCE_FULL) != 0;
    opt.record_worst_case = (flags & CBG_FWD_RECORD_WORST_CASE) != 0;
    r->last = L.forward(to_tensor(x, L.spec.in_channels, L.in_h, L.in_w), up, opt);
    if (eff_ops) *eff_ops = r->last.eff_ops;
  });
}
int ref_conv_dims(void* h, int* oh, int* ow) {
  auto* r = static_cast<RefConv*>(h);
  *oh = r->layer.out_h;
  *ow = r->layer.out_w;
  return CBG_OK;
}
int ref_conv_read_output(void* h, float* y) {
  put_tensor(static_cast<RefConv*>(h)->layer.prev_output, y);
  return CBG_OK;
}
int ref_conv_read_state(void* h, float* y) {
  put_tensor(static_cast<RefConv*>(h)->layer.state.state, y);
  return CBG_OK;
}
int ref_conv_read_changes(void* h, uint8_t* map, int32_t* rc, int64_t* n) {
  auto* r = static_cast<RefConv*>(h);
  if (map) std::memcpy(map, r->last.out_map.bits.data(), r->last.out_map.bits.size());
  if (rc) put_idx(r->last.indexes, rc);
  *n = static_cast<int64_t>(r->last.indexes.size());
  return CBG_OK;
}
int ref_conv_read_worst_case(void* h, uint8_t* map, int64_t* n) {
  auto* r = static_cast<RefConv*>(h);
  if (map && !r->last.worst_case_map.bits.empty())
    std::memcpy(map, r->last.worst_case_map.bits.data(), r->last.worst_case_map.bits.size());
  *n = r->last.propagated_px;
  return CBG_OK;
}
int ref_conv_set_tau(void* h, float tau) {
  static_cast<RefConv*>(h)->layer.tau = tau;
  return CBG_OK;
}

// CBPoolLayer, layers.cpp:133-179
int ref_pool_create(int size, int stride, int c, int in_h, int in_w, int oh, int ow, void** out) {
  return guard([&] { *out = new RefPool{CBPoolLayer(size, stride, c, in_h, in_w, oh, ow), {}}; });
}
void ref_pool_destroy(void* h) { delete static_cast<RefPool*>(h); }
int ref_pool_forward(void* h, const float* x, const uint8_t* up_map, const int32_t* up_rc,
                     int64_t up_n, int force) {
  auto* r = static_cast<RefPool*>(h);
  return guard([&] {
    CBPoolLayer& L = r->layer;
    ChangeMap m;
    IndexList idx;
    UpstreamChange up;
    if (up_map) {
      m = to_map(up_map, L.in_h, L.in_w);
      up.map = &m;
    }
    if (up_rc) {
      idx = to_idx(up_rc, up_n);
      up.indexes = &idx;
    }
    r->last = L.forward(to_tensor(x, L.channels, L.in_h, L.in_w), up, force != 0);
  });
}
int ref_pool_read_output(void* h, float* y) {
  put_tensor(static_cast<RefPool*>(h)->layer.prev_output, y);
  return CBG_OK;
}
int ref_pool_read_changes(void* h, uint8_t* map, int32_t* rc, int64_t* n) {
  auto* r = static_cast<RefPool*>(h);
  if (map) std::memcpy(map, r->last.out_map.bits.data(), r->last.out_map.bits.size());
  if (rc) put_idx(r->last.indexes, rc);
  *n = static_cast<int64_t>(r->last.indexes.size());
  return CBG_OK;
}

// ---- network -------------------------------------------------------------------
// build_network + convert_to_cb, network.cpp:135-137,416-503
int ref_net_create(const cbg_network_spec* n, const float* taus, int n_taus, const int* pol,
                   int mode, void** out) {
  return guard([&] {
    auto r = std::make_unique<RefNet>();
    r->dense = std::make_unique<DenseNetwork>(to_network(*n));
    std::vector<float> t(taus, taus + n_taus);
    std::vector<DetectionPolicy> p;
    if (pol)
      for (int i = 0; i < n_taus; ++i) p.push_back(static_cast<DetectionPolicy>(pol[i]));
    r->cb = convert_to_cb(*r->dense, t, pol ? &p : nullptr, static_cast<DetectMode>(mode));
    *out = r.release();
  });
}
void ref_net_destroy(void* h) { delete static_cast<RefNet*>(h); }
int ref_net_clone(void* h, void** out) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] {
    auto c = std::make_unique<RefNet>();
    c->dense = std::make_unique<DenseNetwork>(*r->dense);
    c->cb = r->cb;
    *out = c.release();
  });
}
int ref_net_node_count(void* h) { return static_cast<int>(static_cast<RefNet*>(h)->cb.nodes().size()); }
int ref_net_node_shape(void* h, int i, int* kind, int* c, int* hh, int* ww) {
  const CBNode& n = static_cast<RefNet*>(h)->cb.nodes()[i];
  *kind = static_cast<int>(n.kind);
  *c = n.out_shape.channels;
  *hh = n.out_shape.height;
  *ww = n.out_shape.width;
  return CBG_OK;
}
// forward_frame, network.cpp:309-414
int ref_net_forward(void* h, const float* frame, int record_worst_case) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] {
    Shape3 s = r->cb.input_shape();
    StatsConfig cfg;
    cfg.record_maps = true;
    cfg.record_worst_case = record_worst_case != 0;
    cfg.timing = false;
    r->last = FrameStats{};
    r->cb.forward_frame(to_tensor(frame, s.channels, s.height, s.width), cfg, &r->last);
  });
}
int ref_net_reset(void* h) {
  static_cast<RefNet*>(h)->cb.reset();
  return CBG_OK;
}
int ref_net_set_thresholds(void* h, const float* taus, int n) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] { r->cb.set_thresholds(std::vector<float>(taus, taus + n)); });
}
int ref_net_read_output(void* h, int node, float* y) {
  auto* r = static_cast<RefNet*>(h);
  const auto& nodes = r->cb.nodes();
  const CBNode& n = nodes[node < 0 ? nodes.size() - 1 : node];
  const Tensor3& t = n.kind == LayerKind::Conv   ? n.conv.prev_output
                     : n.kind == LayerKind::Pool ? n.pool.prev_output
                                                 : n.prev_output;
  put_tensor(t, y);
  return CBG_OK;
}
int ref_net_read_state(void* h, int node, float* y) {
  const CBNode& n = static_cast<RefNet*>(h)->cb.nodes()[node];
  put_tensor(n.conv.state.state, y);
  return CBG_OK;
}
// per node: changed_px, eff_ops, propagated_px; map (out frame) and worst-case map
int ref_net_read_stats(void* h, int node, int64_t* changed, int64_t* eff_ops, int64_t* prop,
                       uint8_t* map, uint8_t* worst) {
  auto* r = static_cast<RefNet*>(h);
  const LayerFrameStats& l = r->last.layers[node];
  if (changed) *changed = l.changed_px;
  if (eff_ops) *eff_ops = l.eff_ops;
  if (prop) *prop = l.propagated_px;
  if (map && !l.map.bits.empty()) std::memcpy(map, l.map.bits.data(), l.map.bits.size());
  if (worst && !l.worst_case_map.bits.empty())
    std::memcpy(worst, l.worst_case_map.bits.data(), l.worst_case_map.bits.size());
  return CBG_OK;
}
// DenseNetwork::forward_all, network.cpp:139-188 (row index = spec row, incl. Act rows)
int ref_dense_forward_row(void* h, const float* frame, int row, float* y) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] {
    const NetworkSpec& s = r->dense->spec();
    std::vector<Tensor3> all =
        r->dense->forward_all(to_tensor(frame, s.in_channels, s.in_height, s.in_width));
    put_tensor(all[row < 0 ? all.size() - 1 : row], y);
  });
}

// ---- calibration (calibration.cpp:95-180) ---------------------------------------
namespace {
std::vector<EvalSequence> to_sequences(const RefNet& r, const cbg_eval_sequence* seqs, int n_seqs) {
  const Shape3 in = r.cb.input_shape();
  const auto& nodes = r.cb.nodes();
  const Shape3 out = nodes.back().out_shape;
  std::vector<EvalSequence> v(n_seqs);
  for (int q = 0; q < n_seqs; ++q) {
    const size_t fe = static_cast<size_t>(in.channels) * in.height * in.width;
    const size_t re = static_cast<size_t>(seqs[q].ref_channels) * out.height * out.width;
    for (int t = 0; t < seqs[q].n_frames; ++t) {
      v[q].frames.push_back(to_tensor(seqs[q].frames + t * fe, in.channels, in.height, in.width));
      v[q].reference.push_back(to_tensor(seqs[q].references + t * re, seqs[q].ref_channels, out.height, out.width));
    }
  }
  return v;
}
}  // namespace

int ref_select_thresholds(void* h, const cbg_eval_sequence* seqs, int n_seqs, const cbg_calib_config* c,
                          float* taus_out, uint8_t* cap_out, cbg_calib_trace_point* trace_out, int trace_cap,
                          int* trace_len) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] {
    CalibConfig cfg;
    cfg.initial_tau = c->initial_tau;
    cfg.growth_factor = c->growth_factor;
    cfg.per_layer_budget = c->per_layer_budget;
    if (c->budget_overrides)
      cfg.budget_overrides.assign(c->budget_overrides, c->budget_overrides + c->n_budget_overrides);
    cfg.metric = static_cast<LossMetric>(c->metric);
    cfg.aggregation = static_cast<LossAggregation>(c->aggregation);
    cfg.max_steps = c->max_steps;
    CalibResult res = select_thresholds(r->cb, to_sequences(*r, seqs, n_seqs), cfg);
    std::copy(res.taus.begin(), res.taus.end(), taus_out);
    for (size_t i = 0; i < res.hit_cap.size(); ++i) cap_out[i] = res.hit_cap[i] ? 1 : 0;
    const int n = std::min<int>(static_cast<int>(res.trace.size()), trace_cap);
    for (int i = 0; i < n; ++i) trace_out[i] = {res.trace[i].layer, res.trace[i].tau, res.trace[i].loss};
    *trace_len = static_cast<int>(res.trace.size());
  });
}

int ref_sweep_threshold_factor(void* h, const float* base_tau, int n_tau, const double* factors, int n_factors,
                               const cbg_eval_sequence* seqs, int n_seqs, int metric, cbg_tradeoff_row* rows) {
  auto* r = static_cast<RefNet*>(h);
  return guard([&] {
    auto curve = sweep_threshold_factor(r->cb, std::vector<float>(base_tau, base_tau + n_tau),
                                        std::vector<double>(factors, factors + n_factors),
                                        to_sequences(*r, seqs, n_seqs), static_cast<LossMetric>(metric));
    for (size_t i = 0; i < curve.size(); ++i)
      rows[i] = {curve[i].factor, curve[i].loss, curve[i].total_eff_ops, curve[i].wall_ns};
  });
}

}  // extern "C"
