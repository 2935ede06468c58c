// ref_stats_csv.cpp — TEST INFRASTRUCTURE ONLY (oracle/_ref/ref_stats_csv).
//
// Prints the reference's forward_sequence + write_stats_csv (network.cpp:505-525,
// io.cpp:660-672) for the scene-labeling net (make_seg7_spec's layers at derived
// dims, io.cpp:605-617; weights fill_random_weights(seed), io.cpp:554-566) on a
// gen_synthetic sequence (io.cpp:499-552), timing off (wall_ns 0). With
// with_reference = 1 the per-frame loss is the MSE against the reference's own
// dense outputs (make_reference, calibration.cpp:55-60).
//
//   ref_stats_csv seed H W tau1..tau5 n_frames n_objects object_size vy vx noise synth_seed with_reference
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <vector>

#include "cbi/calibration.hpp"
#include "cbi/io.hpp"
#include "cbi/network.hpp"

int main(int argc, char** argv) {
  if (argc != 17) {
    std::fprintf(stderr, "usage: ref_stats_csv seed H W tau1..tau5 n_frames n_objects object_size vy vx noise seed ref\n");
    return 2;
  }
  using namespace cbi;
  const unsigned seed = static_cast<unsigned>(std::atoi(argv[1]));
  NetworkSpec spec = make_seg7_spec(seed);
  spec.in_height = std::atoi(argv[2]);
  spec.in_width = std::atoi(argv[3]);
  for (LayerDesc& d : spec.layers) {
    d.conv.out_h = d.conv.out_w = 0;
    d.pool_out_h = d.pool_out_w = 0;
  }
  fill_random_weights(spec, seed);
  std::vector<float> taus;
  for (int i = 0; i < 5; ++i) taus.push_back(static_cast<float>(std::atof(argv[4 + i])));
  SyntheticConfig sc;
  sc.height = spec.in_height;
  sc.width = spec.in_width;
  sc.channels = spec.in_channels;
  sc.n_frames = std::atoi(argv[9]);
  sc.n_objects = std::atoi(argv[10]);
  sc.object_size = std::atoi(argv[11]);
  sc.velocity_y = std::atoi(argv[12]);
  sc.velocity_x = std::atoi(argv[13]);
  sc.noise_std = static_cast<float>(std::atof(argv[14]));
  sc.seed = static_cast<unsigned>(std::atoi(argv[15]));
  const bool with_ref = std::atoi(argv[16]) != 0;
  DenseNetwork dense = build_network(spec);
  CBNetwork net = convert_to_cb(dense, taus);
  const std::vector<Tensor3> frames = gen_synthetic(sc);
  std::vector<Tensor3> ref;
  if (with_ref) ref = make_reference(dense, frames);
  StatsConfig cfg;
  cfg.timing = false;
  SequenceResult res = forward_sequence(net, frames, with_ref ? &ref : nullptr, LossMetric::Mse, cfg);
  write_stats_csv(std::cout, res.stats);
  return 0;
}
