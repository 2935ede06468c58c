// api.cpp — extern "C" entry points of libcbg (include/cbg.h).
// Each entry point catches every exception at the boundary and converts it to
// a status code + thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "runtime.hpp"

namespace cbg {
int conv_gemm_read_trace(unsigned long long* host, int n);
void gen_synthetic(const cbg_synthetic_config& cfg, float* frames, int32_t* corners);
void fill_random_weights(const cbg_network_spec& spec, uint32_t seed, float* const* weights, float* const* biases);
}  // namespace cbg

using cbg::Error;
using cbg::Net;

struct cbg_ctx_s {
  cbg::Ctx ctx;
  explicit cbg_ctx_s(int dev) : ctx(dev) {}
};
struct cbg_net_s {
  cbg_ctx ctx = nullptr;
  std::unique_ptr<Net> net;
};
struct cbg_conv_s {
  cbg_ctx ctx = nullptr;
  std::unique_ptr<Net> net;  // node 0 = external producer, node 1 = the conv
  int in_c = 0, in_h = 0, in_w = 0, out_h = 0, out_w = 0, policy = 0;
  int64_t ops_per_pixel = 0;
  bool had_up_map = false;
  bool forwarded = false;
  unsigned last_flags = 0;
};
struct cbg_pool_s {
  cbg_ctx ctx = nullptr;
  std::unique_ptr<Net> net;
  int channels = 0, in_h = 0, in_w = 0, out_h = 0, out_w = 0;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return CBG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return CBG_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CBG_ERR_CUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) cbg::throw_invalid(std::string(what) + ": null argument");
}
}  // namespace

extern "C" {

const char* cbg_last_error(void) { return g_err.c_str(); }
int cbg_abi_version(void) { return CBG_ABI_VERSION; }

int cbg_device_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
  return p.major == 10 ? 1 : 0;
}

int cbg_ctx_create(int device, cbg_ctx* out) {
  return guard([&] {
    need(out, "cbg_ctx_create");
    *out = new cbg_ctx_s(device);
  });
}
void cbg_ctx_destroy(cbg_ctx ctx) { delete ctx; }
int cbg_ctx_sync(cbg_ctx ctx) {
  return guard([&] {
    need(ctx, "cbg_ctx_sync");
    cbg::cuda_check(cudaStreamSynchronize(ctx->ctx.stream), "cudaStreamSynchronize");
    cbg::cuda_check(cudaStreamSynchronize(ctx->ctx.d2h), "cudaStreamSynchronize");
  });
}
void* cbg_ctx_stream(cbg_ctx ctx) { return ctx ? static_cast<void*>(ctx->ctx.stream) : nullptr; }

int cbg_gen_synthetic(const cbg_synthetic_config* cfg, float* frames_out, int32_t* corners_out) {
  return guard([&] {
    need(cfg, "cbg_gen_synthetic");
    need(frames_out, "cbg_gen_synthetic");
    cbg::gen_synthetic(*cfg, frames_out, corners_out);
  });
}

int cbg_fill_random_weights(const cbg_network_spec* spec, uint32_t seed, float* const* weights,
                            float* const* biases) {
  return guard([&] {
    need(spec, "cbg_fill_random_weights");
    cbg::fill_random_weights(*spec, seed, weights, biases);
  });
}

// ---- network ----------------------------------------------------------------------
int cbg_net_validate(const cbg_network_spec* spec, const float* taus, int n_taus, const int* policies, int mode) {
  return guard([&] {
    need(spec, "cbg_net_validate");
    cbg::convert(*spec, taus, n_taus, policies, mode);
  });
}

int cbg_net_create(cbg_ctx ctx, const cbg_network_spec* spec, const float* taus, int n_taus, const int* policies,
                   int mode, int n_streams, cbg_net* out) {
  return guard([&] {
    need(ctx, "cbg_net_create");
    need(spec, "cbg_net_create");
    need(out, "cbg_net_create");
    auto topo = cbg::convert(*spec, taus, n_taus, policies, mode);
    auto h = std::make_unique<cbg_net_s>();
    h->ctx = ctx;
    h->net = std::make_unique<Net>(&ctx->ctx, std::move(topo), n_streams);
    *out = h.release();
  });
}
void cbg_net_destroy(cbg_net net) { delete net; }

int cbg_net_clone(cbg_net net, cbg_net* out) {
  return guard([&] {
    need(net, "cbg_net_clone");
    need(out, "cbg_net_clone");
    auto h = std::make_unique<cbg_net_s>();
    h->ctx = net->ctx;
    h->net = net->net->clone();
    *out = h.release();
  });
}

int cbg_net_node_count(cbg_net net, int* n) {
  return guard([&] {
    need(net, "cbg_net_node_count");
    *n = static_cast<int>(net->net->nodes().size());
  });
}
int cbg_net_stream_count(cbg_net net, int* n) {
  return guard([&] {
    need(net, "cbg_net_stream_count");
    *n = net->net->streams();
  });
}

int cbg_net_node_info(cbg_net net, int node, cbg_node_info* info) {
  return guard([&] {
    need(net, "cbg_net_node_info");
    need(info, "cbg_net_node_info");
    const auto& nodes = net->net->nodes();
    if (node < 0 || node >= static_cast<int>(nodes.size())) cbg::throw_invalid("node out of range");
    const cbg::NodeDesc& d = nodes[node].d;
    std::memset(info, 0, sizeof(*info));
    info->kind = d.kind;
    std::strncpy(info->name, d.name.c_str(), sizeof(info->name) - 1);
    info->n_inputs = static_cast<int>(d.inputs.size());
    for (int k = 0; k < info->n_inputs && k < 8; ++k) info->inputs[k] = d.inputs[k];
    info->out_channels = d.C;
    info->out_height = d.H;
    info->out_width = d.W;
    info->in_channels = d.Ci;
    info->in_height = d.Hi;
    info->in_width = d.Wi;
    info->policy = d.policy;
    info->fuse_relu = d.relu ? 1 : 0;
    info->tau = d.tau;
    if (d.kind == CBG_LAYER_CONV)
      info->ops_per_pixel = 2ll * d.conv.out_channels * d.conv.in_channels * d.conv.kernel_h * d.conv.kernel_w;
  });
}

int cbg_net_forward(cbg_net net, const float* frames, unsigned flags) {
  return guard([&] {
    need(net, "cbg_net_forward");
    net->net->forward(frames, flags);
  });
}
int cbg_net_forward_u8(cbg_net net, const uint8_t* frames_hwc, unsigned flags) {
  return guard([&] {
    need(net, "cbg_net_forward_u8");
    net->net->forward_u8(frames_hwc, flags);
  });
}
int cbg_net_set_stream_thresholds(cbg_net net, int stream, const float* taus, int n_taus) {
  return guard([&] {
    need(net, "cbg_net_set_stream_thresholds");
    if (n_taus > 0) need(taus, "cbg_net_set_stream_thresholds");
    net->net->set_stream_thresholds(stream, std::vector<float>(taus, taus + std::max(0, n_taus)));
  });
}
int cbg_select_thresholds(cbg_net proto, const cbg_eval_sequence* seqs, int n_seqs, const cbg_calib_config* cfg,
                          float* taus_out, uint8_t* hit_cap_out, cbg_calib_trace_point* trace_out, int trace_cap,
                          int* trace_len) {
  return guard([&] {
    need(proto, "cbg_select_thresholds");
    need(cfg, "cbg_select_thresholds");
    need(taus_out, "cbg_select_thresholds");
    std::vector<float> taus;
    std::vector<uint8_t> cap;
    std::vector<cbg_calib_trace_point> trace;
    cbg::select_thresholds(&proto->ctx->ctx, proto->net->topology(), seqs, n_seqs, *cfg, taus, cap, trace);
    std::copy(taus.begin(), taus.end(), taus_out);
    if (hit_cap_out) std::copy(cap.begin(), cap.end(), hit_cap_out);
    const int n = std::min<int>(static_cast<int>(trace.size()), std::max(0, trace_cap));
    if (trace_out) std::copy(trace.begin(), trace.begin() + n, trace_out);
    if (trace_len) *trace_len = static_cast<int>(trace.size());
  });
}
int cbg_sweep_threshold_factor(cbg_net proto, const float* base_tau, int n_tau, const double* factors,
                               int n_factors, const cbg_eval_sequence* seqs, int n_seqs, int metric,
                               cbg_tradeoff_row* rows_out) {
  return guard([&] {
    need(proto, "cbg_sweep_threshold_factor");
    if (n_tau > 0) need(base_tau, "cbg_sweep_threshold_factor");
    if (n_factors > 0) {
      need(factors, "cbg_sweep_threshold_factor");
      need(rows_out, "cbg_sweep_threshold_factor");
    }
    std::vector<cbg_tradeoff_row> rows;
    cbg::sweep_threshold_factor(&proto->ctx->ctx, proto->net->topology(),
                                std::vector<float>(base_tau, base_tau + std::max(0, n_tau)),
                                std::vector<double>(factors, factors + std::max(0, n_factors)), seqs, n_seqs, metric,
                                rows);
    std::copy(rows.begin(), rows.end(), rows_out);
  });
}
int cbg_net_reset(cbg_net net, int stream) {
  return guard([&] {
    need(net, "cbg_net_reset");
    net->net->reset(stream);
  });
}
int cbg_net_set_thresholds(cbg_net net, const float* taus, int n_taus) {
  return guard([&] {
    need(net, "cbg_net_set_thresholds");
    if (n_taus > 0) need(taus, "cbg_net_set_thresholds");
    net->net->set_thresholds(std::vector<float>(taus, taus + n_taus));
  });
}
int cbg_net_thresholds(cbg_net net, float* taus, int n_taus) {
  return guard([&] {
    need(net, "cbg_net_thresholds");
    auto t = net->net->thresholds();
    if (n_taus < static_cast<int>(t.size())) cbg::throw_invalid("cbg_net_thresholds: buffer too small");
    std::copy(t.begin(), t.end(), taus);
  });
}
int cbg_net_set_dense(cbg_net net, int dense) {
  return guard([&] {
    need(net, "cbg_net_set_dense");
    net->net->set_dense(dense != 0);
  });
}

int cbg_net_read_output(cbg_net net, int node, int stream, float* out_chw) {
  return guard([&] {
    need(net, "cbg_net_read_output");
    need(out_chw, "cbg_net_read_output");
    net->net->read_output(node, stream, out_chw);
  });
}
int cbg_net_read_state(cbg_net net, int node, int stream, float* out_chw) {
  return guard([&] {
    need(net, "cbg_net_read_state");
    need(out_chw, "cbg_net_read_state");
    net->net->read_state(node, stream, out_chw);
  });
}
int cbg_net_read_changes(cbg_net net, int node, int stream, uint8_t* map_out, int32_t* rowcol_out,
                         int64_t* count_out) {
  return guard([&] {
    need(net, "cbg_net_read_changes");
    net->net->read_changes(node, stream, map_out, rowcol_out, count_out, false);
  });
}
int cbg_net_read_worst_case(cbg_net net, int node, int stream, uint8_t* map_out, int64_t* count_out) {
  return guard([&] {
    need(net, "cbg_net_read_worst_case");
    const auto& nodes = net->net->nodes();
    if (node < 0 || node >= static_cast<int>(nodes.size()) || nodes[node].d.kind != CBG_LAYER_CONV)
      cbg::throw_invalid("worst-case maps exist for conv nodes only");
    if (!net->net->has_worst_case(node)) {
      if (count_out) *count_out = -1;
      return;
    }
    net->net->read_changes(node, stream, map_out, nullptr, count_out, true);
  });
}
int cbg_net_read_stats(cbg_net net, int stream, cbg_layer_stats* stats, int n_nodes) {
  return guard([&] {
    need(net, "cbg_net_read_stats");
    need(stats, "cbg_net_read_stats");
    Net& n = *net->net;
    const int nn = static_cast<int>(n.nodes().size());
    if (n_nodes < nn) cbg::throw_invalid("cbg_net_read_stats: buffer too small");
    if (stream < 0 || stream >= n.streams()) cbg::throw_invalid("stream out of range");
    std::vector<int32_t> counts;
    n.read_counts(counts);
    for (int i = 0; i < nn; ++i) {
      const cbg::NodeDesc& d = n.nodes()[i].d;
      cbg_layer_stats& s = stats[i];
      s.changed_px = n.count_of(counts, i, stream);
      s.total_px = static_cast<int64_t>(d.H) * d.W;
      s.eff_ops = 0;
      s.propagated_px = -1;
      if (d.kind == CBG_LAYER_CONV) {
        s.eff_ops = 2ll * d.conv.out_channels * d.conv.in_channels * d.conv.kernel_h * d.conv.kernel_w * s.changed_px;
        if (n.has_worst_case(i))
          s.propagated_px = d.inputs[0] >= 0 ? n.count_of(counts, i, stream, true) : s.changed_px;
      }
    }
  });
}
int cbg_net_read_counts(cbg_net net, int64_t* counts_out) {
  return guard([&] {
    need(net, "cbg_net_read_counts");
    need(counts_out, "cbg_net_read_counts");
    Net& n = *net->net;
    std::vector<int32_t> counts;
    n.read_counts(counts);
    const int nn = static_cast<int>(n.nodes().size()), S = n.streams();
    for (int i = 0; i < nn; ++i)
      for (int s = 0; s < S; ++s) counts_out[static_cast<size_t>(i) * S + s] = n.count_of(counts, i, s);
  });
}

int cbg_net_last_launches(cbg_net net, int* launches) {
  return guard([&] {
    need(net, "cbg_net_last_launches");
    *launches = net->net->last_launches();
  });
}
int cbg_net_set_kernel_timing(cbg_net net, int enabled) {
  return guard([&] {
    need(net, "cbg_net_set_kernel_timing");
    net->net->set_timing(enabled != 0);
  });
}
int cbg_net_timing_report(cbg_net net, char* buf, int len) {
  return guard([&] {
    need(net, "cbg_net_timing_report");
    need(buf, "cbg_net_timing_report");
    const std::string js = net->net->timing_report();
    if (static_cast<int>(js.size()) + 1 > len) cbg::throw_invalid("cbg_net_timing_report: buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
  });
}
int cbg_net_copy_output_async(cbg_net net, int node, void* host_dst) {
  return guard([&] {
    need(net, "cbg_net_copy_output_async");
    need(host_dst, "cbg_net_copy_output_async");
    net->net->copy_output_async(node, host_dst);
  });
}
int cbg_net_copy_counts_async(cbg_net net, int32_t* host_dst, int32_t* node_slot) {
  return guard([&] {
    need(net, "cbg_net_copy_counts_async");
    if (node_slot)
      for (size_t i = 0; i < net->net->nodes().size(); ++i) node_slot[i] = net->net->node_slot(static_cast<int>(i));
    if (host_dst) net->net->copy_counts_async(host_dst);
  });
}
int cbg_net_kernel_labels(cbg_net net, unsigned flags, char* buf, int len) {
  return guard([&] {
    need(net, "cbg_net_kernel_labels");
    need(buf, "cbg_net_kernel_labels");
    std::string js = "[";
    for (const std::string& l : net->net->kernel_labels(flags)) js += (js.size() > 1 ? ", \"" : "\"") + l + "\"";
    js += "]";
    if (static_cast<int>(js.size()) >= len) cbg::throw_invalid("cbg_net_kernel_labels: buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
  });
}
int cbg_ctx_set_persistent_sms(cbg_ctx ctx, int sms) {
  return guard([&] {
    need(ctx, "cbg_ctx_set_persistent_sms");
    if (sms < 0) cbg::throw_invalid("cbg_ctx_set_persistent_sms: negative SM count");
    ctx->ctx.persistent_sms = sms;
  });
}
int cbg_net_detect_slots(cbg_net net, int32_t* det_slot) {
  return guard([&] {
    need(net, "cbg_net_detect_slots");
    need(det_slot, "cbg_net_detect_slots");
    for (size_t i = 0; i < net->net->nodes().size(); ++i) det_slot[i] = net->net->det_slot(static_cast<int>(i));
  });
}
int cbg_debug_gemm_trace(unsigned long long* buf, int n) { return cbg::conv_gemm_read_trace(buf, n); }
int cbg_net_count_slots(cbg_net net, int* slots) {
  return guard([&] {
    need(net, "cbg_net_count_slots");
    *slots = std::max(1, net->net->count_slots());
  });
}
int cbg_host_alloc(int64_t bytes, void** ptr) {
  return guard([&] {
    need(ptr, "cbg_host_alloc");
    if (bytes < 0) cbg::throw_invalid("cbg_host_alloc: negative size");
    *ptr = nullptr;
    cbg::cuda_check(cudaHostAlloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 1)),
                                  cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc");
  });
}
void cbg_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}
int cbg_net_output_delta_bytes(cbg_net net, int node, int64_t* bytes) {
  return guard([&] {
    need(net, "cbg_net_output_delta_bytes");
    need(bytes, "cbg_net_output_delta_bytes");
    *bytes = static_cast<int64_t>(net->net->output_delta_bytes(node));
  });
}
int cbg_net_last_delta_dma_bytes(cbg_net net, int64_t* bytes) {
  return guard([&] {
    need(net, "cbg_net_last_delta_dma_bytes");
    need(bytes, "cbg_net_last_delta_dma_bytes");
    *bytes = static_cast<int64_t>(net->net->last_delta_dma_bytes());
  });
}
int cbg_net_copy_output_delta(cbg_net net, int node, void* host_buf) {
  return guard([&] {
    need(net, "cbg_net_copy_output_delta");
    need(host_buf, "cbg_net_copy_output_delta");
    net->net->copy_output_delta(node, host_buf);
  });
}
int cbg_net_apply_output_delta(cbg_net net, int node, const void* host_buf, float* mirror, int stream_begin,
                               int stream_end) {
  return guard([&] {
    need(net, "cbg_net_apply_output_delta");
    need(host_buf, "cbg_net_apply_output_delta");
    need(mirror, "cbg_net_apply_output_delta");
    net->net->apply_output_delta(node, host_buf, mirror, stream_begin, stream_end);
  });
}
int cbg_net_copy_output_detached(cbg_net net, int node, void* host_dst) {
  return guard([&] {
    need(net, "cbg_net_copy_output_detached");
    need(host_dst, "cbg_net_copy_output_detached");
    net->net->copy_output_detached(node, host_dst);
  });
}
void* cbg_ctx_copy_stream(cbg_ctx ctx) { return ctx ? static_cast<void*>(ctx->ctx.d2h) : nullptr; }
int cbg_net_output_bytes(cbg_net net, int node, int64_t* bytes) {
  return guard([&] {
    need(net, "cbg_net_output_bytes");
    const auto& nodes = net->net->nodes();
    if (node < 0) node = static_cast<int>(nodes.size()) - 1;
    if (node >= static_cast<int>(nodes.size())) cbg::throw_invalid("bad node");
    *bytes = static_cast<int64_t>(nodes[node].out.bytes);
  });
}

// ---- standalone conv layer (CBConvLayer, layers.cpp:33-131) -------------------------
int cbg_conv_create(cbg_ctx ctx, const cbg_conv_spec* spec, float tau, int policy, int fuse_relu, int mode, int in_h,
                    int in_w, cbg_conv* out) {
  return guard([&] {
    need(ctx, "cbg_conv_create");
    need(spec, "cbg_conv_create");
    need(out, "cbg_conv_create");
    cbg::ConvDesc c = cbg::conv_from_c(*spec);
    cbg::validate_conv(c);
    if (!(tau >= 0.0f)) cbg::throw_invalid("CBConvLayer: tau must be >= 0");
    if (policy < CBG_POLICY_DETECT || policy > CBG_POLICY_REUSE1X1) cbg::throw_invalid("unknown policy");
    if (mode != CBG_MODE_CLOSEDLOOP && mode != CBG_MODE_FEEDFORWARD) cbg::throw_invalid("unknown detect mode");
    if (in_h < 1 || in_w < 1) cbg::throw_invalid("CBConvLayer: input dims must be >= 1");
    const int oh = cbg::conv_out_dim(in_h, c.kernel_h, c.stride, c.padding, c.out_h);
    const int ow = cbg::conv_out_dim(in_w, c.kernel_w, c.stride, c.padding, c.out_w);
    if (policy == CBG_POLICY_REUSE1X1 &&
        !(c.kernel_h == 1 && c.kernel_w == 1 && c.stride == 1 && oh == in_h && ow == in_w))
      cbg::throw_config("reuse_1x1 policy requires a 1x1 stride-1 shape-preserving layer");
    cbg::Topology topo;
    topo.C = c.in_channels;
    topo.H = in_h;
    topo.W = in_w;
    topo.mode = mode;
    cbg::NodeDesc ext;
    ext.kind = cbg::kExternal;
    ext.name = "input";
    ext.C = ext.Ci = c.in_channels;
    ext.H = ext.Hi = in_h;
    ext.W = ext.Wi = in_w;
    cbg::NodeDesc conv;
    conv.kind = CBG_LAYER_CONV;
    conv.name = "conv";
    conv.inputs = {0};
    conv.C = c.out_channels;
    conv.H = oh;
    conv.W = ow;
    conv.Ci = c.in_channels;
    conv.Hi = in_h;
    conv.Wi = in_w;
    conv.tau = tau;
    conv.policy = policy;
    conv.relu = fuse_relu != 0;
    conv.conv = c;
    topo.nodes = {ext, conv};
    auto h = std::make_unique<cbg_conv_s>();
    h->ctx = ctx;
    h->in_c = c.in_channels;
    h->in_h = in_h;
    h->in_w = in_w;
    h->out_h = oh;
    h->out_w = ow;
    h->policy = policy;
    h->ops_per_pixel = 2ll * c.out_channels * c.in_channels * c.kernel_h * c.kernel_w;
    h->net = std::make_unique<Net>(&ctx->ctx, std::move(topo), 1);
    *out = h.release();
  });
}
void cbg_conv_destroy(cbg_conv layer) { delete layer; }
int cbg_conv_out_dims(cbg_conv layer, int* out_h, int* out_w) {
  return guard([&] {
    need(layer, "cbg_conv_out_dims");
    *out_h = layer->out_h;
    *out_w = layer->out_w;
  });
}

int cbg_conv_forward(cbg_conv layer, const float* x, const uint8_t* up_map, const int32_t* up_rowcol, int64_t up_count,
                     unsigned flags, int64_t* eff_ops_out) {
  return guard([&] {
    need(layer, "cbg_conv_forward");
    need(x, "cbg_conv_forward");
    const bool full = (flags & CBG_FWD_FORCE_FULL) != 0;
    if (!full) {  // layers.cpp:80-99
      if (layer->policy == CBG_POLICY_PROPAGATE && !up_map)
        cbg::throw_config("propagate policy requires an upstream change map");
      if (layer->policy == CBG_POLICY_REUSE1X1 && (!up_map || !up_rowcol))
        cbg::throw_config("reuse_1x1 policy requires upstream map and indexes");
    }
    if (up_rowcol)
      for (int64_t k = 0; k < up_count; ++k)
        if (up_rowcol[2 * k] < 0 || up_rowcol[2 * k] >= layer->in_h || up_rowcol[2 * k + 1] < 0 ||
            up_rowcol[2 * k + 1] >= layer->in_w)
          cbg::throw_invalid("update_output: index outside the output tensor");
    layer->net->set_external(x, up_map, up_rowcol, up_count, full);
    layer->had_up_map = up_map != nullptr;
    layer->last_flags = flags;
    layer->net->forward(nullptr, flags & (CBG_FWD_FORCE_FULL | CBG_FWD_RECORD_WORST_CASE));
    layer->forwarded = true;
    if (eff_ops_out) {
      std::vector<int32_t> counts;
      layer->net->read_counts(counts);
      *eff_ops_out = layer->ops_per_pixel * layer->net->count_of(counts, 1, 0);
    }
  });
}
int cbg_conv_read_output(cbg_conv layer, float* out_chw) {
  return guard([&] {
    need(layer, "cbg_conv_read_output");
    layer->net->read_output(1, 0, out_chw);
  });
}
int cbg_conv_read_state(cbg_conv layer, float* out_chw) {
  return guard([&] {
    need(layer, "cbg_conv_read_state");
    layer->net->read_state(1, 0, out_chw);
  });
}
int cbg_conv_read_changes(cbg_conv layer, uint8_t* map_out, int32_t* rowcol_out, int64_t* count_out) {
  return guard([&] {
    need(layer, "cbg_conv_read_changes");
    layer->net->read_changes(1, 0, map_out, rowcol_out, count_out, false);
  });
}
int cbg_conv_read_worst_case(cbg_conv layer, uint8_t* map_out, int64_t* count_out) {
  return guard([&] {
    need(layer, "cbg_conv_read_worst_case");
    if (!(layer->last_flags & CBG_FWD_RECORD_WORST_CASE)) {
      if (count_out) *count_out = -1;
      return;
    }
    // layers.cpp:108-117: without an upstream map the detected set is its own worst case
    layer->net->read_changes(1, 0, map_out, nullptr, count_out, layer->had_up_map);
  });
}
int cbg_conv_set_tau(cbg_conv layer, float tau) {
  return guard([&] {
    need(layer, "cbg_conv_set_tau");
    layer->net->set_thresholds({tau});
  });
}

// ---- standalone pool layer (CBPoolLayer, layers.cpp:133-179) --------------------------
int cbg_pool_create(cbg_ctx ctx, int size, int stride, int channels, int in_h, int in_w, int out_h, int out_w,
                    cbg_pool* out) {
  return guard([&] {
    need(ctx, "cbg_pool_create");
    need(out, "cbg_pool_create");
    if (size < 1 || stride < 1) cbg::throw_invalid("CBPoolLayer: size/stride must be >= 1");
    if ((out_h - 1) * stride >= in_h || (out_w - 1) * stride >= in_w || out_h < 1 || out_w < 1)
      cbg::throw_invalid("CBPoolLayer: output dims leave an empty window");
    if (channels < 1) cbg::throw_invalid("CBPoolLayer: channels must be >= 1");
    cbg::Topology topo;
    topo.C = channels;
    topo.H = in_h;
    topo.W = in_w;
    cbg::NodeDesc ext;
    ext.kind = cbg::kExternal;
    ext.name = "input";
    ext.C = ext.Ci = channels;
    ext.H = ext.Hi = in_h;
    ext.W = ext.Wi = in_w;
    cbg::NodeDesc pool;
    pool.kind = CBG_LAYER_POOL;
    pool.name = "pool";
    pool.inputs = {0};
    pool.C = pool.Ci = channels;
    pool.H = out_h;
    pool.W = out_w;
    pool.Hi = in_h;
    pool.Wi = in_w;
    pool.pool_size = size;
    pool.pool_stride = stride;
    topo.nodes = {ext, pool};
    auto h = std::make_unique<cbg_pool_s>();
    h->ctx = ctx;
    h->channels = channels;
    h->in_h = in_h;
    h->in_w = in_w;
    h->out_h = out_h;
    h->out_w = out_w;
    h->net = std::make_unique<Net>(&ctx->ctx, std::move(topo), 1);
    *out = h.release();
  });
}
void cbg_pool_destroy(cbg_pool layer) { delete layer; }
int cbg_pool_forward(cbg_pool layer, const float* x, const uint8_t* up_map, const int32_t* up_rowcol, int64_t up_count,
                     int force_full_update) {
  return guard([&] {
    need(layer, "cbg_pool_forward");
    need(x, "cbg_pool_forward");
    if (!force_full_update && !up_map) cbg::throw_config("change-based pooling requires an upstream change map");
    layer->net->set_external(x, up_map, up_rowcol, up_count);
    layer->net->forward(nullptr, force_full_update ? CBG_FWD_FORCE_FULL : 0u);
  });
}
int cbg_pool_read_output(cbg_pool layer, float* out_chw) {
  return guard([&] {
    need(layer, "cbg_pool_read_output");
    layer->net->read_output(1, 0, out_chw);
  });
}
int cbg_pool_read_changes(cbg_pool layer, uint8_t* map_out, int32_t* rowcol_out, int64_t* count_out) {
  return guard([&] {
    need(layer, "cbg_pool_read_changes");
    layer->net->read_changes(1, 0, map_out, rowcol_out, count_out, false);
  });
}

}  // extern "C"
