// ref_bench.cpp — TEST/BASELINE INFRASTRUCTURE ONLY (oracle). Never part of the product.
//
// Times the UNMODIFIED reference (cbi, compiled from /root/reference/proj/src by
// oracle/Makefile) on the host cores: one cbi::CBNetwork per std::thread, one camera
// stream per network ("multiple camera streams = multiple CBNetwork
// instances"; the reference has no mutable globals, so this is safe). Used by
// bench.py's cpu_baseline leg and `bench.py --impl reference`.
//
// Workload = the scene-labeling net of make_seg7_spec (io.cpp:568-617) with
// derived (unpinned) dims at the requested resolution, weights from
// fill_random_weights(seed 1) (io.cpp:554-566), stream s fed by
// gen_synthetic{seed = 1000 + s} (io.cpp:499-552). The bootstrap frame is
// excluded from timing, as in SURVEY.md §8(d) / BASELINE.md §4.
//
// Output: one JSON object on stdout.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cbi/io.hpp"
#include "cbi/network.hpp"

using namespace cbi;

namespace {

NetworkSpec seg_spec(int h, int w) {
  NetworkSpec spec;
  spec.in_channels = 3;
  spec.in_height = h;
  spec.in_width = w;
  auto conv = [](const char* name, int in, int out, int k, int pad, bool relu) {
    LayerDesc d;
    d.kind = LayerKind::Conv;
    d.name = name;
    d.conv.in_channels = in;
    d.conv.out_channels = out;
    d.conv.kernel_h = d.conv.kernel_w = k;
    d.conv.padding = pad;
    d.fuse_relu = relu;
    return d;
  };
  auto act = [](const char* name) {
    LayerDesc d;
    d.kind = LayerKind::Act;
    d.name = name;
    return d;
  };
  auto pool = [](const char* name) {
    LayerDesc d;
    d.kind = LayerKind::Pool;
    d.name = name;
    d.pool_size = 2;
    d.pool_stride = 2;
    return d;
  };
  spec.layers.push_back(conv("L1", 3, 16, 7, 0, false));
  spec.layers.push_back(act("L2a"));
  spec.layers.push_back(pool("L2b"));
  spec.layers.push_back(conv("L3", 16, 64, 7, 3, false));
  spec.layers.push_back(act("L4a"));
  spec.layers.push_back(pool("L4b"));
  spec.layers.push_back(conv("L5", 64, 256, 7, 3, true));
  spec.layers.push_back(conv("L6", 256, 64, 1, 0, true));
  spec.layers.push_back(conv("L7", 64, 8, 1, 0, false));
  fill_random_weights(spec, 1);
  return spec;
}

int arg_int(int argc, char** argv, const char* key, int def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], key) == 0) return std::atoi(argv[i + 1]);
  return def;
}
double arg_dbl(int argc, char** argv, const char* key, double def) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], key) == 0) return std::atof(argv[i + 1]);
  return def;
}
bool has_flag(int argc, char** argv, const char* key) {
  for (int i = 1; i < argc; ++i)
    if (std::strcmp(argv[i], key) == 0) return true;
  return false;
}

}  // namespace

int main(int argc, char** argv) {
  const int h = arg_int(argc, argv, "--height", 480);
  const int w = arg_int(argc, argv, "--width", 640);
  const int streams = arg_int(argc, argv, "--streams", 1);
  int threads = arg_int(argc, argv, "--threads", 0);
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  threads = std::min(threads, streams);
  const int frames = arg_int(argc, argv, "--frames", 4);  // timed frames per stream (max)
  const int n_objects = arg_int(argc, argv, "--objects", 4);
  const int object_size = arg_int(argc, argv, "--object-size", 32);
  const int velocity = arg_int(argc, argv, "--velocity", 4);
  const double noise = arg_dbl(argc, argv, "--noise", 0.0);
  const double tau = arg_dbl(argc, argv, "--tau", 0.05);
  const double budget_s = arg_dbl(argc, argv, "--time-budget", 20.0);
  const bool dense = has_flag(argc, argv, "--dense");
  // --pnm8: frames as a PNM sequence would deliver them (bench.py's workload):
  // byte = floor(clamp(v, 0, 1) * 255 + 0.5), then load_pnm's byte / 255.0f
  const bool pnm8 = has_flag(argc, argv, "--pnm8");

  NetworkSpec spec = seg_spec(h, w);
  DenseNetwork net = build_network(spec);
  CBNetwork proto = convert_to_cb(net, std::vector<float>(5, static_cast<float>(tau)));

  std::vector<std::vector<Tensor3>> seqs(streams);
  for (int s = 0; s < streams; ++s) {
    SyntheticConfig cfg;
    cfg.height = h;
    cfg.width = w;
    cfg.channels = 3;
    cfg.n_frames = frames + 1;
    cfg.n_objects = n_objects;
    cfg.object_size = object_size;
    cfg.velocity_y = cfg.velocity_x = velocity;
    cfg.noise_std = static_cast<float>(noise);
    cfg.seed = 1000u + static_cast<unsigned>(s);
    seqs[s] = gen_synthetic(cfg);
    if (pnm8)
      for (Tensor3& f : seqs[s])
        for (float& v : f.data) {
          const float q = std::floor(std::min(std::max(v, 0.0f), 1.0f) * 255.0f + 0.5f);
          v = static_cast<float>(static_cast<unsigned char>(q)) / 255.0f;
        }
  }

  std::vector<CBNetwork> nets(streams, proto);
  // Bootstrap (untimed): frame 0 of every stream.
  {
    std::vector<std::thread> pool;
    std::atomic<int> next{0};
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (int s = next++; s < streams; s = next++) {
          if (!dense) nets[s].forward_frame(seqs[s][0], StatsConfig{false, false, false, false});
        }
      });
    for (auto& th : pool) th.join();
  }

  // Timed: frames 1..F round-robin, stopping when the time budget is spent.
  std::atomic<long long> done{0};
  std::atomic<long long> changed_l1{0};
  const auto t0 = std::chrono::steady_clock::now();
  const auto deadline = t0 + std::chrono::duration<double>(budget_s);
  {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        for (int f = 1; f <= frames; ++f) {
          for (int s = t; s < streams; s += threads) {
            if (std::chrono::steady_clock::now() > deadline) return;
            if (dense) {
              net.forward(seqs[s][f]);
            } else {
              FrameStats fs;
              nets[s].forward_frame(seqs[s][f], StatsConfig{false, false, false, false}, &fs);
              changed_l1 += fs.layers[0].changed_px;
            }
            ++done;
          }
        }
      });
    for (auto& th : pool) th.join();
  }
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const double l1_px = static_cast<double>(net.topology().shape[0].pixels());
  const double frac = done > 0 ? static_cast<double>(changed_l1) / (done * l1_px) : 0.0;
  std::printf(
      "{\"frames\": %lld, \"seconds\": %.6f, \"fps\": %.6f, \"threads\": %d, \"streams\": %d, "
      "\"height\": %d, \"width\": %d, \"dense\": %s, \"l1_change_frac\": %.6f}\n",
      static_cast<long long>(done), secs, secs > 0 ? done / secs : 0.0, threads, streams, h, w,
      dense ? "true" : "false", frac);
  return 0;
}
