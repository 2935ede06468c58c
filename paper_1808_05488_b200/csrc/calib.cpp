// calib.cpp — threshold calibration on the GPU (calibration.cpp:68-180).
//
// The reference's calibration replays whole sequences through a CBNetwork for
// every candidate threshold vector, one after the other, on one core. Here a
// stream set of the hot path evaluates many threshold vectors at once: stream k
// of a set replays the same frames (CBG_FWD_BROADCAST_INPUT) under its own
// thresholds (Net::set_stream_thresholds). The selection rules, the losses and
// the trace follow the reference exactly; only the outputs they are computed
// from come from the B200 path (fp32-accurate).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "runtime.hpp"

namespace cbg {

namespace {

// argmax over channels, first maximum wins (calibration.cpp:11-22)
int argmax_channel(const float* t, int C, size_t HW, size_t p) {
  int best = 0;
  float best_v = t[p];
  for (int c = 1; c < C; ++c) {
    const float v = t[static_cast<size_t>(c) * HW + p];
    if (v > best_v) {
      best_v = v;
      best = c;
    }
  }
  return best;
}

// loss_value (calibration.cpp:51-53): Mse (calibration.cpp:41-49) or
// 1 - pixel_accuracy (calibration.cpp:26-39). pred is CHW [C][H][W].
double loss_value(int metric, const float* pred, int C, int H, int W, const float* ref, int ref_c) {
  const size_t HW = static_cast<size_t>(H) * W;
  if (metric == CBG_LOSS_MSE) {
    if (ref_c != C) throw_invalid("mse: shapes differ");
    double acc = 0.0;
    const size_t n = static_cast<size_t>(C) * HW;
    for (size_t i = 0; i < n; ++i) {
      const double d = static_cast<double>(pred[i]) - ref[i];
      acc += d * d;
    }
    return acc / static_cast<double>(n);
  }
  if (ref_c != 1 && ref_c != C) throw_invalid("pixel_accuracy: reference channels must be 1 (labels) or match");
  int64_t hits = 0;
  for (size_t p = 0; p < HW; ++p) {
    const int a = argmax_channel(pred, C, HW, p);
    const int r = ref_c == 1 ? static_cast<int>(ref[p]) : argmax_channel(ref, ref_c, HW, p);
    hits += a == r;
  }
  return 1.0 - static_cast<double>(hits) / static_cast<double>(HW);
}

struct Shapes {
  int C, H, W;        // network input
  int Co, Ho, Wo;     // network output (last node)
  size_t in_elems, out_elems;
};

Shapes shapes_of(const Topology& t) {
  Shapes s{};
  s.C = t.C, s.H = t.H, s.W = t.W;
  const NodeDesc& last = t.nodes.back();
  s.Co = last.C, s.Ho = last.H, s.Wo = last.W;
  s.in_elems = static_cast<size_t>(s.C) * s.H * s.W;
  s.out_elems = static_cast<size_t>(s.Co) * s.Ho * s.Wo;
  return s;
}

int conv_count(const Topology& t) {
  int n = 0;
  for (const NodeDesc& d : t.nodes) n += d.kind == CBG_LAYER_CONV;
  return n;
}

void check_sequences(const cbg_eval_sequence* seqs, int n_seqs, const char* who) {
  if (n_seqs < 1 || seqs == nullptr) throw_invalid(std::string(who) + ": no evaluation sequences");
  for (int q = 0; q < n_seqs; ++q)
    if (seqs[q].n_frames < 1 || !seqs[q].frames || !seqs[q].references)
      throw_invalid(std::string(who) + ": sequence needs frames and per-frame references");
}

// Replays `seq` from reset on every stream of `net` (stream k under taus[k]);
// calls on_frame(t, outputs [S][Co][Ho][Wo] host, counts) after every frame if
// per_frame, else once after the last frame.
template <class F>
void replay(Net& net, const Shapes& sh, const cbg_eval_sequence& seq, const std::vector<std::vector<float>>& taus,
            bool per_frame, F&& on_frame) {
  const int S = net.streams();
  for (int k = 0; k < S; ++k) net.set_stream_thresholds(k, taus[k]);
  net.reset(-1);
  std::vector<float> out(static_cast<size_t>(S) * sh.out_elems);
  std::vector<int32_t> counts;
  const int last = static_cast<int>(net.nodes().size()) - 1;
  for (int t = 0; t < seq.n_frames; ++t) {
    net.forward(seq.frames + static_cast<size_t>(t) * sh.in_elems, CBG_FWD_BROADCAST_INPUT);
    if (per_frame || t == seq.n_frames - 1) {
      for (int k = 0; k < S; ++k) net.read_output(last, k, out.data() + static_cast<size_t>(k) * sh.out_elems);
      net.read_counts(counts);
      on_frame(t, out, counts);
    }
  }
}

}  // namespace

void select_thresholds(Ctx* ctx, const Topology& topo, const cbg_eval_sequence* seqs, int n_seqs,
                       const cbg_calib_config& cfg, std::vector<float>& taus, std::vector<uint8_t>& hit_cap,
                       std::vector<cbg_calib_trace_point>& trace) {
  // argument checks in the reference's order (calibration.cpp:97-107)
  if (!(cfg.initial_tau > 0.0)) throw_invalid("calibration: initial_tau must be > 0");
  if (!(cfg.growth_factor > 1.0)) throw_invalid("calibration: growth_factor must be > 1");
  if (cfg.per_layer_budget < 0.0) throw_invalid("calibration: per_layer_budget must be >= 0");
  if (cfg.max_steps < 1) throw_invalid("calibration: max_steps must be >= 1");
  if (n_seqs < 1 || seqs == nullptr) throw_invalid("calibration: no evaluation sequences");
  const int n_conv = conv_count(topo);
  if (cfg.n_budget_overrides > 0 && cfg.n_budget_overrides != n_conv)
    throw_invalid("calibration: budget override count != conv layer count");
  check_sequences(seqs, n_seqs, "calibration");
  if (cfg.metric != CBG_LOSS_MSE && cfg.metric != CBG_LOSS_PIXEL_ACCURACY_DELTA) throw_invalid("unknown loss metric");
  const Shapes sh = shapes_of(topo);

  // one stream set per sequence: stream 0 = the current vector (base loss),
  // stream 1 + k = candidate k (initial_tau * growth^k)
  const int S = cfg.max_steps + 1;
  std::vector<std::unique_ptr<Net>> nets;
  for (int q = 0; q < n_seqs; ++q) nets.push_back(std::make_unique<Net>(ctx, topo, S));
  std::vector<double> cand(cfg.max_steps);
  {
    double tau = cfg.initial_tau;
    for (int k = 0; k < cfg.max_steps; ++k, tau *= cfg.growth_factor) cand[k] = tau;
  }

  taus.assign(n_conv, 0.0f);
  hit_cap.assign(n_conv, 0);
  trace.clear();
  for (int layer = 0; layer < n_conv; ++layer) {
    const double budget = cfg.n_budget_overrides > 0 ? cfg.budget_overrides[layer] : cfg.per_layer_budget;
    std::vector<std::vector<float>> vecs(S, taus);
    for (int k = 0; k < cfg.max_steps; ++k) vecs[1 + k][layer] = static_cast<float>(cand[k]);
    // eval_taus (calibration.cpp:68-90): final-frame loss per sequence, aggregated
    std::vector<double> mean(S, 0.0), worst(S, 0.0);
    for (int q = 0; q < n_seqs; ++q) {
      replay(*nets[q], sh, seqs[q], vecs, false, [&](int, const std::vector<float>& out, const std::vector<int32_t>&) {
        const float* ref = seqs[q].references +
                           static_cast<size_t>(seqs[q].n_frames - 1) * seqs[q].ref_channels * sh.Ho * sh.Wo;
        for (int k = 0; k < S; ++k) {
          const double l = loss_value(cfg.metric, out.data() + static_cast<size_t>(k) * sh.out_elems, sh.Co, sh.Ho,
                                      sh.Wo, ref, seqs[q].ref_channels);
          mean[k] += l;
          worst[k] = std::max(worst[k], l);
        }
      });
    }
    auto agg = [&](int k) {
      return cfg.aggregation == CBG_AGG_MEAN ? mean[k] / static_cast<double>(n_seqs) : worst[k];
    };
    const double base_loss = agg(0);
    float selected = 0.0f;
    bool capped = true;
    for (int k = 0; k < cfg.max_steps; ++k) {
      const double loss = agg(1 + k);
      trace.push_back({layer, cand[k], loss});
      if (loss - base_loss > budget) {
        capped = false;
        break;
      }
      selected = static_cast<float>(cand[k]);
    }
    taus[layer] = selected;
    hit_cap[layer] = capped ? 1 : 0;
  }
}

void sweep_threshold_factor(Ctx* ctx, const Topology& topo, const std::vector<float>& base_tau,
                            const std::vector<double>& factors, const cbg_eval_sequence* seqs, int n_seqs, int metric,
                            std::vector<cbg_tradeoff_row>& rows) {
  // argument checks in the reference's order (calibration.cpp:148-156)
  if (static_cast<int>(base_tau.size()) != conv_count(topo)) throw_invalid("sweep: expected one base tau per conv layer");
  for (size_t i = 0; i < factors.size(); ++i) {
    if (factors[i] < 0.0) throw_invalid("sweep: factors must be >= 0");
    if (i > 0 && factors[i] <= factors[i - 1]) throw_invalid("sweep: factors must be strictly increasing");
  }
  if (n_seqs < 1 || seqs == nullptr) throw_invalid("sweep: no evaluation sequences");
  check_sequences(seqs, n_seqs, "sweep");
  if (metric != CBG_LOSS_MSE && metric != CBG_LOSS_PIXEL_ACCURACY_DELTA) throw_invalid("unknown loss metric");
  rows.assign(factors.size(), cbg_tradeoff_row{});
  if (factors.empty()) return;
  const Shapes sh = shapes_of(topo);
  const int S = static_cast<int>(factors.size());
  std::vector<std::vector<float>> vecs(S, std::vector<float>(base_tau.size()));
  for (int k = 0; k < S; ++k)
    for (size_t i = 0; i < base_tau.size(); ++i) vecs[k][i] = static_cast<float>(factors[k] * base_tau[i]);
  std::vector<int> conv_nodes;
  std::vector<int64_t> ops_pp;
  for (size_t i = 0; i < topo.nodes.size(); ++i) {
    const NodeDesc& d = topo.nodes[i];
    if (d.kind != CBG_LAYER_CONV) continue;
    conv_nodes.push_back(static_cast<int>(i));
    ops_pp.push_back(2ll * d.conv.out_channels * d.conv.in_channels * d.conv.kernel_h * d.conv.kernel_w);
  }
  std::vector<double> loss_sum(S, 0.0);
  std::vector<int64_t> loss_n(S, 0);
  Net net(ctx, topo, S);
  for (int q = 0; q < n_seqs; ++q) {
    const auto t0 = std::chrono::steady_clock::now();
    replay(net, sh, seqs[q], vecs, true, [&](int t, const std::vector<float>& out, const std::vector<int32_t>& counts) {
      if (t < 1) return;  // FrameStats.frame < 2: the bootstrap frame (calibration.cpp:170)
      const float* ref = seqs[q].references + static_cast<size_t>(t) * seqs[q].ref_channels * sh.Ho * sh.Wo;
      for (int k = 0; k < S; ++k) {
        loss_sum[k] += loss_value(metric, out.data() + static_cast<size_t>(k) * sh.out_elems, sh.Co, sh.Ho, sh.Wo, ref,
                                  seqs[q].ref_channels);
        ++loss_n[k];
        for (size_t c = 0; c < conv_nodes.size(); ++c)
          rows[k].total_eff_ops += ops_pp[c] * net.count_of(counts, conv_nodes[c], k);
      }
    });
    const int64_t ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    for (int k = 0; k < S; ++k) rows[k].wall_ns += ns / S;
  }
  for (int k = 0; k < S; ++k) {
    rows[k].factor = factors[k];
    rows[k].loss = loss_n[k] > 0 ? loss_sum[k] / static_cast<double>(loss_n[k]) : 0.0;
  }
}

}  // namespace cbg
