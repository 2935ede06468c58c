// synth.cpp — deterministic synthetic inputs, host side.
//
// Mirrors the reference's harness generators so the B200 path can be fed the
// exact sequences the CPU reference sees (tests check byte equality against the
// reference build):
//   gen_synthetic        reference io.cpp:499-552 (seeded static background,
//                        bouncing solid rectangles, optional Gaussian noise)
//   fill_random_weights  reference io.cpp:554-566 (He-uniform weights)
// The generator is std::mt19937 driven directly with fixed transforms
// (reference DetRng, io.cpp:461-484), so outputs are platform-independent.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "runtime.hpp"

namespace cbg {
namespace {

class SeededRng {
 public:
  explicit SeededRng(uint32_t seed) : eng_(seed) {}
  // 24-bit uniform in [0, 1)
  float uniform() { return static_cast<float>((eng_() >> 8) * (1.0 / 16777216.0)); }
  int below(int n) { return n > 0 ? static_cast<int>(eng_() % static_cast<uint32_t>(n)) : 0; }
  // Box-Muller pair, the second value cached for the next call
  float normal() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    const double u1 = (static_cast<double>(eng_() >> 8) + 0.5) / 16777216.0;
    const double u2 = static_cast<double>(eng_() >> 8) / 16777216.0;
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 6.283185307179586 * u2;
    cache_ = static_cast<float>(rad * std::sin(ang));
    cached_ = true;
    return static_cast<float>(rad * std::cos(ang));
  }

 private:
  std::mt19937 eng_;
  bool cached_ = false;
  float cache_ = 0.0f;
};

// Advance one coordinate; reflect at the borders (io.cpp:486-495).
int step_bounce(int pos, int& vel, int size, int limit) {
  int next = pos + vel;
  if (next < 0 || next + size > limit) {
    vel = -vel;
    next = std::min(std::max(pos + vel, 0), limit - size);
  }
  return next;
}

}  // namespace

void gen_synthetic(const cbg_synthetic_config& cfg, float* frames, int32_t* corners) {
  if (cfg.height < 1 || cfg.width < 1 || cfg.channels < 1 || cfg.n_frames < 1)
    throw_invalid("gen_synthetic: dims, channels and n_frames must be >= 1");
  if (cfg.n_objects < 0 || cfg.noise_std < 0.0f) throw_invalid("gen_synthetic: n_objects and noise_std must be >= 0");
  if (cfg.n_objects > 0 && (cfg.object_size < 1 || cfg.object_size > cfg.height || cfg.object_size > cfg.width))
    throw_invalid("gen_synthetic: objects must fit in the frame");
  SeededRng rng(cfg.seed);
  const size_t plane = static_cast<size_t>(cfg.height) * cfg.width;
  const size_t fsize = plane * cfg.channels;
  std::vector<float> bg(fsize);
  for (float& v : bg) v = rng.uniform();

  struct Obj {
    std::vector<float> color;
    int row, col, vy, vx;
  };
  std::vector<Obj> objs(cfg.n_objects);
  for (int k = 0; k < cfg.n_objects; ++k) {
    Obj& o = objs[k];
    o.color.resize(cfg.channels);
    for (float& c : o.color) c = rng.uniform();
    o.row = rng.below(cfg.height - cfg.object_size + 1);
    o.col = rng.below(cfg.width - cfg.object_size + 1);
    const int dir = (k % 2 == 0) ? 1 : -1;
    o.vy = dir * cfg.velocity_y;
    o.vx = dir * cfg.velocity_x;
  }
  for (int t = 0; t < cfg.n_frames; ++t) {
    float* f = frames + static_cast<size_t>(t) * fsize;
    std::memcpy(f, bg.data(), fsize * sizeof(float));
    for (int k = 0; k < cfg.n_objects; ++k) {
      const Obj& o = objs[k];
      if (corners) {
        corners[(static_cast<size_t>(t) * cfg.n_objects + k) * 2] = o.row;
        corners[(static_cast<size_t>(t) * cfg.n_objects + k) * 2 + 1] = o.col;
      }
      for (int c = 0; c < cfg.channels; ++c)
        for (int j = o.row; j < o.row + cfg.object_size; ++j)
          for (int i = o.col; i < o.col + cfg.object_size; ++i) f[c * plane + static_cast<size_t>(j) * cfg.width + i] = o.color[c];
    }
    if (cfg.noise_std > 0.0f)
      for (size_t v = 0; v < fsize; ++v) f[v] += cfg.noise_std * rng.normal();
    for (Obj& o : objs) {
      o.row = step_bounce(o.row, o.vy, cfg.object_size, cfg.height);
      o.col = step_bounce(o.col, o.vx, cfg.object_size, cfg.width);
    }
  }
}

void fill_random_weights(const cbg_network_spec& spec, uint32_t seed, float* const* weights, float* const* biases) {
  SeededRng rng(seed);
  int k = 0;
  for (int i = 0; i < spec.n_layers; ++i) {
    const cbg_layer_desc& d = spec.layers[i];
    if (d.kind != CBG_LAYER_CONV) continue;
    const cbg_conv_spec& c = d.conv;
    const float fan_in = static_cast<float>(c.in_channels) * c.kernel_h * c.kernel_w;
    const float a = std::sqrt(6.0f / fan_in);
    const size_t nw = static_cast<size_t>(c.out_channels) * c.in_channels * c.kernel_h * c.kernel_w;
    for (size_t w = 0; w < nw; ++w) weights[k][w] = (rng.uniform() * 2.0f - 1.0f) * a;
    for (int b = 0; b < c.out_channels; ++b) biases[k][b] = (rng.uniform() * 2.0f - 1.0f) * 0.05f;
    ++k;
  }
}

}  // namespace cbg
