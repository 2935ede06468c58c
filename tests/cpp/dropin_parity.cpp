// dropin_parity.cpp — TEST: the C++ drop-in (include/cbg/cbi_gpu.hpp, namespace cbg)
// used exactly like the reference API (namespace cbi), on identical inputs.
// Links the unmodified reference objects (oracle/_ref) as the checker.
//
// Exit 0 = parity holds: layer-1 change maps/index lists bit-exact every frame,
// final map max_rel_err <= 1e-4 (tests/oracles.hpp:59-66 metric), identical
// changed_px per node, and the reference error categories on bad wiring.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <vector>

#include "cbg/cbi_gpu.hpp"
#include "cbi/io.hpp"
#include "cbi/calibration.hpp"
#include "cbi/network.hpp"

namespace {
double max_rel_err(const std::vector<float>& a, const std::vector<float>& b) {
  double w = 0.0;
  for (size_t i = 0; i < a.size(); ++i)
    w = std::max(w, std::fabs(double(a[i]) - b[i]) / std::max(1.0, std::fabs(double(b[i]))));
  return w;
}

// the same NetworkSpec in both namespaces (reference make_seg7_spec layer list, derived dims)
template <class NS, class LD, class LK>
NS seg_spec(const cbi::NetworkSpec& ref) {
  NS s;
  s.in_channels = ref.in_channels;
  s.in_height = ref.in_height;
  s.in_width = ref.in_width;
  for (const cbi::LayerDesc& d : ref.layers) {
    LD l;
    l.kind = static_cast<LK>(static_cast<int>(d.kind));
    l.name = d.name;
    l.from = d.from;
    l.conv.in_channels = d.conv.in_channels;
    l.conv.out_channels = d.conv.out_channels;
    l.conv.kernel_h = d.conv.kernel_h;
    l.conv.kernel_w = d.conv.kernel_w;
    l.conv.stride = d.conv.stride;
    l.conv.padding = d.conv.padding;
    l.conv.out_h = d.conv.out_h;
    l.conv.out_w = d.conv.out_w;
    l.conv.weights = d.conv.weights;
    l.conv.bias = d.conv.bias;
    l.fuse_relu = d.fuse_relu;
    l.pool_size = d.pool_size;
    l.pool_stride = d.pool_stride;
    l.pool_out_h = d.pool_out_h;
    l.pool_out_w = d.pool_out_w;
    s.layers.push_back(l);
  }
  return s;
}
}  // namespace

int main() {
  int bad = 0;
  // reference topology at 96x128 with derived dims (drop the pinned out dims)
  cbi::NetworkSpec rspec = cbi::make_seg7_spec(1);
  rspec.in_height = 96;
  rspec.in_width = 128;
  for (cbi::LayerDesc& d : rspec.layers) {
    d.conv.out_h = d.conv.out_w = 0;
    d.pool_out_h = d.pool_out_w = 0;
  }
  const std::vector<float> taus(5, 0.05f);
  cbi::SyntheticConfig sc;
  sc.height = 96;
  sc.width = 128;
  sc.channels = 3;
  sc.n_frames = 6;
  sc.n_objects = 3;
  sc.object_size = 12;
  sc.velocity_y = sc.velocity_x = 3;
  sc.seed = 77;
  const std::vector<cbi::Tensor3> frames = cbi::gen_synthetic(sc);

  cbi::CBNetwork ref = cbi::convert_to_cb(cbi::build_network(rspec), taus);
  cbg::CBNetwork gpu = cbg::convert_to_cb(
      cbg::build_network(seg_spec<cbg::NetworkSpec, cbg::LayerDesc, cbg::LayerKind>(rspec)), taus);

  for (size_t t = 0; t < frames.size(); ++t) {
    cbi::StatsConfig rc;
    rc.record_maps = true;
    rc.timing = false;
    cbi::FrameStats rfs;
    const cbi::Tensor3& want = ref.forward_frame(frames[t], rc, &rfs);
    cbg::Tensor3 x(frames[t].channels, frames[t].height, frames[t].width);
    x.data = frames[t].data;
    cbg::StatsConfig gc;
    gc.record_maps = true;
    cbg::FrameStats gfs;
    const cbg::Tensor3& got = gpu.forward_frame(x, gc, &gfs);
    const double err = max_rel_err(got.data, want.data);
    if (err > 1e-4) {
      std::printf("frame %zu: max_rel_err %.3g\n", t, err);
      ++bad;
    }
    if (gfs.layers[0].map.bits != rfs.layers[0].map.bits) {
      std::printf("frame %zu: layer-1 map differs\n", t);
      ++bad;
    }
    for (size_t i = 0; i < rfs.layers.size(); ++i)
      if (gfs.layers[i].changed_px != rfs.layers[i].changed_px || gfs.layers[i].eff_ops != rfs.layers[i].eff_ops) {
        std::printf("frame %zu node %zu: changed_px %lld vs %lld\n", t, i, (long long)gfs.layers[i].changed_px,
                    (long long)rfs.layers[i].changed_px);
        ++bad;
      }
  }

  // error categories (network.cpp:416-503)
  try {
    cbg::convert_to_cb(cbg::build_network(seg_spec<cbg::NetworkSpec, cbg::LayerDesc, cbg::LayerKind>(rspec)),
                       std::vector<float>(4, 0.0f));
    ++bad;
  } catch (const cbg::InvalidInputError&) {
  }
  try {
    std::vector<cbg::DetectionPolicy> pol(5, cbg::DetectionPolicy::Detect);
    pol[0] = cbg::DetectionPolicy::Propagate;
    cbg::convert_to_cb(cbg::build_network(seg_spec<cbg::NetworkSpec, cbg::LayerDesc, cbg::LayerKind>(rspec)),
                       taus, &pol);
    ++bad;
  } catch (const cbg::ConfigError&) {
  }
  // calibration (calibration.cpp:95-141): the drop-in's GPU select_thresholds
  // against the reference's on the same sequences and dense references
  {
    cbi::DenseNetwork dense = cbi::build_network(rspec);
    std::vector<cbi::EvalSequence> rseqs(2);
    std::vector<cbg::EvalSequence> gseqs(2);
    for (int q = 0; q < 2; ++q) {
      cbi::SyntheticConfig c2 = sc;
      c2.n_frames = 4;
      c2.seed = 300 + q;
      c2.noise_std = 0.01f;
      rseqs[q].frames = cbi::gen_synthetic(c2);
      rseqs[q].reference = cbi::make_reference(dense, rseqs[q].frames);
      for (size_t t = 0; t < rseqs[q].frames.size(); ++t) {
        const cbi::Tensor3& f = rseqs[q].frames[t];
        const cbi::Tensor3& r = rseqs[q].reference[t];
        cbg::Tensor3 gf(f.channels, f.height, f.width), gr(r.channels, r.height, r.width);
        gf.data = f.data;
        gr.data = r.data;
        gseqs[q].frames.push_back(gf);
        gseqs[q].reference.push_back(gr);
      }
    }
    cbi::CalibConfig rc;
    rc.initial_tau = 0.01;
    rc.growth_factor = 2.0;
    rc.per_layer_budget = 1e-3;
    rc.max_steps = 6;
    cbg::CalibConfig gc;
    gc.initial_tau = rc.initial_tau;
    gc.growth_factor = rc.growth_factor;
    gc.per_layer_budget = rc.per_layer_budget;
    gc.max_steps = rc.max_steps;
    const cbi::CalibResult want = cbi::select_thresholds(ref, rseqs, rc);
    const cbg::CalibResult got = cbg::select_thresholds(gpu, gseqs, gc);
    if (got.taus != want.taus || got.trace.size() != want.trace.size()) {
      std::printf("select_thresholds differs\n");
      ++bad;
    }
    for (size_t i = 0; i < std::min(got.trace.size(), want.trace.size()); ++i)
      if (got.trace[i].tau != want.trace[i].tau ||
          std::abs(got.trace[i].loss - want.trace[i].loss) > 1e-3 * std::abs(want.trace[i].loss) + 1e-9) {
        std::printf("trace %zu: tau %g/%g loss %g/%g\n", i, got.trace[i].tau, want.trace[i].tau, got.trace[i].loss,
                    want.trace[i].loss);
        ++bad;
      }
  }
  // forward_sequence + write_stats_csv (io.cpp:660-672): byte-identical with timing off
  {
    cbi::CBNetwork r2 = cbi::convert_to_cb(cbi::build_network(rspec), taus);
    cbg::CBNetwork g2 = cbg::convert_to_cb(
        cbg::build_network(seg_spec<cbg::NetworkSpec, cbg::LayerDesc, cbg::LayerKind>(rspec)), taus);
    cbi::StatsConfig rc;
    rc.timing = false;
    std::vector<cbg::Tensor3> gframes;
    for (const cbi::Tensor3& f : frames) {
      cbg::Tensor3 x(f.channels, f.height, f.width);
      x.data = f.data;
      gframes.push_back(x);
    }
    std::ostringstream ro, go;
    cbi::write_stats_csv(ro, cbi::forward_sequence(r2, frames, nullptr, cbi::LossMetric::Mse, rc).stats);
    cbg::write_stats_csv(go, cbg::forward_sequence(g2, gframes).stats);
    if (ro.str() != go.str()) {
      std::printf("stats CSV differs:\n%s---\n%s", ro.str().c_str(), go.str().c_str());
      ++bad;
    }
  }
  std::printf("dropin_parity: %s (%d problems)\n", bad ? "FAIL" : "PASS", bad);
  return bad ? 1 : 0;
}
