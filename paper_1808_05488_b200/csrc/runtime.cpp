// runtime.cpp — host runtime of the B200 CBinfer path (see runtime.hpp).
#include "runtime.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <unordered_map>

#include "kernels.hpp"

namespace cbg {

[[noreturn]] void throw_invalid(const std::string& m) { throw Error(CBG_ERR_INVALID_INPUT, m); }
[[noreturn]] void throw_config(const std::string& m) { throw Error(CBG_ERR_CONFIG, m); }
void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) throw Error(CBG_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  throw Error(CBG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// ---- shapes / validation (tensor.cpp:9-43) ------------------------------------
int conv_out_dim(int in_dim, int kernel, int stride, int padding, int pinned) {
  if (pinned > 0) return pinned;
  const int v = (in_dim + 2 * padding - kernel) / stride + 1;
  if (in_dim + 2 * padding - kernel < 0 || v < 1)
    throw_invalid("conv output dim < 1 (input " + std::to_string(in_dim) + ", kernel " + std::to_string(kernel) +
                  ", stride " + std::to_string(stride) + ", padding " + std::to_string(padding) + ")");
  return v;
}

void validate_conv(const ConvDesc& c) {
  if (c.in_channels < 1 || c.out_channels < 1 || c.kernel_h < 1 || c.kernel_w < 1)
    throw_invalid("conv spec: channel and kernel dims must be >= 1");
  if (c.stride < 1) throw_invalid("conv spec: stride must be >= 1");
  if (c.padding < 0) throw_invalid("conv spec: padding must be >= 0");
  if (c.out_h < 0 || c.out_w < 0 || (c.out_h > 0) != (c.out_w > 0))
    throw_invalid("conv spec: explicit output dims must both be set and >= 1");
  const size_t wc = static_cast<size_t>(c.out_channels) * c.in_channels * c.kernel_h * c.kernel_w;
  if (c.weights.size() != wc)
    throw_invalid("conv spec: weight count " + std::to_string(c.weights.size()) + " != out*in*kh*kw = " +
                  std::to_string(wc));
  if (c.bias.size() != static_cast<size_t>(c.out_channels))
    throw_invalid("conv spec: bias count " + std::to_string(c.bias.size()) + " != out_channels = " +
                  std::to_string(c.out_channels));
}

ConvDesc conv_from_c(const cbg_conv_spec& s) {
  ConvDesc c;
  c.in_channels = s.in_channels;
  c.out_channels = s.out_channels;
  c.kernel_h = s.kernel_h;
  c.kernel_w = s.kernel_w;
  c.stride = s.stride;
  c.padding = s.padding;
  c.out_h = s.out_h;
  c.out_w = s.out_w;
  if (s.in_channels > 0 && s.out_channels > 0 && s.kernel_h > 0 && s.kernel_w > 0) {
    const size_t wc = static_cast<size_t>(s.out_channels) * s.in_channels * s.kernel_h * s.kernel_w;
    if (!s.weights || !s.bias) throw_invalid("conv spec: weights and bias must be given");
    c.weights.assign(s.weights, s.weights + wc);
    c.bias.assign(s.bias, s.bias + s.out_channels);
  }
  return c;
}

// ---- resolve + convert_to_cb (network.cpp:37-133, 416-503) ----------------------
namespace {
std::string layer_label(const cbg_layer_desc& d, int i) {
  return (d.name && d.name[0]) ? std::string(d.name) : "L" + std::to_string(i + 1);
}
std::string where_label(const cbg_layer_desc& d, int i) {
  return "layer " + std::to_string(i) + " (" + layer_label(d, i) + ")";
}
int pool_out_dim(int in_dim, int size, int stride, int explicit_dim, const std::string& where) {
  if (explicit_dim > 0) {
    if ((explicit_dim - 1) * stride >= in_dim)
      throw_invalid(where + ": pool output dim " + std::to_string(explicit_dim) + " leaves an empty window");
    return explicit_dim;
  }
  if (in_dim < size) throw_invalid(where + ": pool window larger than input dim " + std::to_string(in_dim));
  return (in_dim - size) / stride + 1;
}
struct Shape {
  int c = 0, h = 0, w = 0;
  bool operator==(const Shape& o) const { return c == o.c && h == o.h && w == o.w; }
};
}  // namespace

Topology convert(const cbg_network_spec& spec, const float* taus, int n_taus, const int* policies, int mode) {
  if (spec.in_channels < 1 || spec.in_height < 1 || spec.in_width < 1)
    throw_invalid("network spec: input resolution must be positive");
  if (spec.n_layers < 1 || spec.layers == nullptr) throw_invalid("network spec: no layers");
  if (mode != CBG_MODE_CLOSEDLOOP && mode != CBG_MODE_FEEDFORWARD) throw_invalid("unknown detect mode");
  const int n = spec.n_layers;
  std::unordered_map<std::string, int> by_name;
  for (int i = 0; i < n; ++i) {
    const cbg_layer_desc& d = spec.layers[i];
    if (!d.name || !d.name[0]) continue;
    const std::string name = d.name;
    if (name == "input" || !by_name.emplace(name, i).second)
      throw_invalid(where_label(d, i) + ": duplicate or reserved name");
  }
  std::vector<std::vector<int>> inputs(n);
  std::vector<Shape> shape(n);
  const Shape in_shape{spec.in_channels, spec.in_height, spec.in_width};
  auto shape_of = [&](int id) { return id < 0 ? in_shape : shape[id]; };
  std::vector<ConvDesc> convs(n);

  for (int i = 0; i < n; ++i) {
    const cbg_layer_desc& d = spec.layers[i];
    const std::string where = where_label(d, i);
    std::vector<int>& in = inputs[i];
    if (d.n_from <= 0) {
      in.push_back(i - 1);
    } else {
      for (int k = 0; k < d.n_from; ++k) {
        const std::string src = d.from[k] ? d.from[k] : "";
        if (src == "input") {
          in.push_back(-1);
          continue;
        }
        auto it = by_name.find(src);
        if (it == by_name.end() || it->second >= i)
          throw_invalid(where + ": unknown or later producer '" + src + "'");
        in.push_back(it->second);
      }
    }
    try {
      switch (d.kind) {
        case CBG_LAYER_CONV: {
          if (in.size() != 1) throw_invalid("conv takes exactly one producer");
          convs[i] = conv_from_c(d.conv);
          validate_conv(convs[i]);
          const Shape s = shape_of(in[0]);
          if (s.c != d.conv.in_channels)
            throw_invalid("expects " + std::to_string(d.conv.in_channels) + " input channels, producer has " +
                          std::to_string(s.c));
          shape[i] = {d.conv.out_channels,
                      conv_out_dim(s.h, d.conv.kernel_h, d.conv.stride, d.conv.padding, d.conv.out_h),
                      conv_out_dim(s.w, d.conv.kernel_w, d.conv.stride, d.conv.padding, d.conv.out_w)};
          break;
        }
        case CBG_LAYER_ACT:
          if (in.size() != 1) throw_invalid("act takes exactly one producer");
          if (!(d.act_slope >= 0.0f) || !std::isfinite(d.act_slope)) throw_invalid("act slope must be >= 0");
          shape[i] = shape_of(in[0]);
          break;
        case CBG_LAYER_UPSAMPLE: {  // extension: nearest-neighbour, integer factor
          if (in.size() != 1) throw_invalid("upsample takes exactly one producer");
          if (d.upsample < 1 || d.upsample > 64) throw_invalid("upsample factor must be in [1, 64]");
          const Shape s = shape_of(in[0]);
          // pool_out_h / pool_out_w > 0: cropped output dims (<= in * factor)
          if (d.pool_out_h < 0 || d.pool_out_w < 0 || d.pool_out_h > s.h * d.upsample || d.pool_out_w > s.w * d.upsample)
            throw_invalid("upsample output dims out of range");
          shape[i] = {s.c, d.pool_out_h > 0 ? d.pool_out_h : s.h * d.upsample,
                      d.pool_out_w > 0 ? d.pool_out_w : s.w * d.upsample};
          break;
        }
        case CBG_LAYER_POOL: {
          if (in.size() != 1) throw_invalid("pool takes exactly one producer");
          if (d.pool_size < 1 || d.pool_stride < 1) throw_invalid("pool size/stride must be >= 1");
          const Shape s = shape_of(in[0]);
          shape[i] = {s.c, pool_out_dim(s.h, d.pool_size, d.pool_stride, d.pool_out_h, "h"),
                      pool_out_dim(s.w, d.pool_size, d.pool_stride, d.pool_out_w, "w")};
          break;
        }
        case CBG_LAYER_ADD: {
          if (in.size() < 2) throw_invalid("add takes at least two producers");
          const Shape s = shape_of(in[0]);
          for (int id : in)
            if (!(shape_of(id) == s)) throw_invalid("add producers differ in shape");
          shape[i] = s;
          break;
        }
        case CBG_LAYER_CONCAT: {
          if (in.size() < 2) throw_invalid("concat takes at least two producers");
          const Shape s = shape_of(in[0]);
          int ch = 0;
          for (int id : in) {
            const Shape si = shape_of(id);
            if (si.h != s.h || si.w != s.w) throw_invalid("concat producers differ in spatial dims");
            ch += si.c;
          }
          shape[i] = {ch, s.h, s.w};
          break;
        }
        default:
          throw_invalid("unknown layer kind " + std::to_string(d.kind));
      }
    } catch (const Error& e) {
      if (e.code != CBG_ERR_INVALID_INPUT) throw;
      throw_invalid(where + ": " + e.what());
    }
  }

  int conv_rows = 0;
  for (int i = 0; i < n; ++i) conv_rows += spec.layers[i].kind == CBG_LAYER_CONV;
  if (n_taus != conv_rows)
    throw_invalid("convert_to_cb: expected " + std::to_string(conv_rows) + " thresholds, got " +
                  std::to_string(n_taus));
  for (int k = 0; k < n_taus; ++k)
    if (!(taus[k] >= 0.0f)) throw_invalid("convert_to_cb: tau must be >= 0");
  if (policies)
    for (int k = 0; k < n_taus; ++k)
      if (policies[k] < CBG_POLICY_DETECT || policies[k] > CBG_POLICY_REUSE1X1) throw_invalid("unknown policy");

  std::vector<int> consumers(n, 0);
  for (int i = 0; i < n; ++i)
    for (int id : inputs[i])
      if (id >= 0) ++consumers[id];

  Topology topo;
  topo.C = spec.in_channels;
  topo.H = spec.in_height;
  topo.W = spec.in_width;
  topo.mode = mode;
  std::vector<int> new_id(n, -1);
  int conv_idx = 0;
  for (int i = 0; i < n; ++i) {
    const cbg_layer_desc& d = spec.layers[i];
    const std::string where = where_label(d, i);
    const Shape ish = shape_of(inputs[i][0]);
    if (d.kind == CBG_LAYER_ACT) {
      const int src = inputs[i][0];
      if (src < 0 || spec.layers[src].kind != CBG_LAYER_CONV)
        throw_config(where + ": standalone activation can only be absorbed into a conv");
      if (consumers[src] != 1) throw_config(where + ": cannot absorb activation, conv output has other consumers");
      topo.nodes[new_id[src]].relu = true;
      topo.nodes[new_id[src]].slope = d.act_slope;
      new_id[i] = new_id[src];
      continue;
    }
    NodeDesc nd;
    nd.kind = d.kind;
    nd.name = layer_label(d, i);
    nd.C = shape[i].c;
    nd.H = shape[i].h;
    nd.W = shape[i].w;
    nd.Ci = ish.c;
    nd.Hi = ish.h;
    nd.Wi = ish.w;
    for (int id : inputs[i]) nd.inputs.push_back(id < 0 ? -1 : new_id[id]);
    if (d.kind == CBG_LAYER_CONV) {
      const int policy = policies ? policies[conv_idx] : CBG_POLICY_DETECT;
      if (policy != CBG_POLICY_DETECT && nd.inputs[0] < 0)
        throw_config(where + ": " + (policy == CBG_POLICY_PROPAGATE ? "propagate" : "reuse_1x1") +
                     " policy needs an upstream change-based layer");
      nd.conv = convs[i];
      nd.tau = taus[conv_idx];
      nd.policy = policy;
      nd.relu = d.fuse_relu != 0;
      nd.slope = d.act_slope;
      if (!(nd.slope >= 0.0f) || !std::isfinite(nd.slope)) throw_invalid(where + ": act slope must be >= 0");
      if (policy == CBG_POLICY_REUSE1X1 &&
          !(nd.conv.kernel_h == 1 && nd.conv.kernel_w == 1 && nd.conv.stride == 1 && nd.H == nd.Hi && nd.W == nd.Wi))
        throw_config(where + ": reuse_1x1 policy requires a 1x1 stride-1 shape-preserving layer");
      ++conv_idx;
    } else if (d.kind == CBG_LAYER_POOL) {
      if (nd.inputs[0] < 0) throw_config(where + ": change-based pooling needs an upstream layer");
      nd.pool_size = d.pool_size;
      nd.pool_stride = d.pool_stride;
    } else if (d.kind == CBG_LAYER_UPSAMPLE) {
      if (nd.inputs[0] < 0) throw_config(where + ": change-based upsampling needs an upstream layer");
      nd.up = d.upsample;
    } else {
      for (int id : nd.inputs)
        if (id < 0) throw_config(where + ": change-based joins need upstream layers, not the input");
      if (nd.inputs.size() > 4) throw Error(CBG_ERR_UNSUPPORTED, where + ": joins support at most 4 producers");
    }
    new_id[i] = static_cast<int>(topo.nodes.size());
    topo.nodes.push_back(std::move(nd));
  }
  return topo;
}

// ---- device resources --------------------------------------------------------------
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    if (p) cudaFree(p);
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}
DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}
void DevBuf::alloc(size_t n) {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = n;
  if (n == 0) return;
  CK(cudaMalloc(&p, n));
  CK(cudaMemset(p, 0, n));
  // the memset runs on the legacy stream, which does not order against the
  // non-blocking ctx streams: finish it before any ctx-stream write can land
  CK(cudaStreamSynchronize(nullptr));
}

Ctx::Ctx(int dev) : device(dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) throw Error(CBG_ERR_UNSUPPORTED, "no CUDA device visible");
  if (dev < 0 || dev >= n) throw_invalid("device index out of range");
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    throw Error(CBG_ERR_UNSUPPORTED, std::string("kernels are built for sm_100a; device is ") + prop.name);
  sm_count = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
}
Ctx::~Ctx() {
  if (d2h) cudaStreamDestroy(d2h);
  if (stream) cudaStreamDestroy(stream);
}

// ---- Net ------------------------------------------------------------------------------
namespace {
int round4(int c) { return (c + 3) & ~3; }

uint32_t tf32_round(float x) {  // round-to-nearest-away into the top 19 bits (cvt.rna.tf32.f32)
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return u & 0xffffe000u;
  u += 0x1000u;
  return u & 0xffffe000u;
}

// Pre-swizzled UMMA SW128 K-major images of the (kj, ki, c)-ordered weight
// matrix, split into tf32 hi / lo: [n_tile][kb][hi|lo][npad rows][128 B].
// IEEE binary16 round-to-nearest-even of a float (normal, subnormal, overflow to inf).
uint16_t f16_rn(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) return static_cast<uint16_t>(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));
  if (ax >= 0x477ff000u) return static_cast<uint16_t>(sign | 0x7c00u);  // rounds to >= 65520: inf
  if (ax < 0x38800000u) {  // below 2^-14: fp16 subnormal (or zero), quantum 2^-24
    const float q = std::ldexp(std::fabs(f), 24);
    const float r = std::nearbyint(q);  // round-half-even under the default rounding mode
    return static_cast<uint16_t>(sign | static_cast<uint32_t>(r));
  }
  uint32_t m = ax + 0xfffu + ((ax >> 13) & 1u);  // round the 13 dropped bits to nearest even
  return static_cast<uint16_t>(sign | ((m - 0x38000000u) >> 13));
}
float f16_to_f32(uint16_t h) {
  const uint32_t sign = (h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  float v;
  if (e == 0) v = std::ldexp(static_cast<float>(m), -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = std::ldexp(static_cast<float>(m | 0x400u), static_cast<int>(e) - 25);
  return sign ? -v : v;
}

// Exponent ew with max|w| * 2^-ew < 2^15 (mirrors f16_scale_exp in conv_tcgen05.cu).
int weight_exp(const std::vector<float>& w) {
  float m = 0.0f;
  for (float v : w) m = std::max(m, std::fabs(v));
  if (!(m > 0.0f) || !std::isfinite(m)) return 0;
  uint32_t u;
  std::memcpy(&u, &m, 4);
  const int e = static_cast<int>((u >> 23) & 0xffu) - 127 - 14;
  return std::min(126, std::max(-126, e));
}

void build_weight_image(const NodeRT& n, std::vector<uint8_t>& img, std::vector<uint32_t>& ktab,
                        std::vector<float>& bias) {
  const ConvDesc& c = n.d.conv;
  const int taps = c.kernel_h * c.kernel_w;
  const int Kreal = taps * n.Csi;
  const bool f16 = n.prec != 0;
  const int Brow = f16 ? 64 : 128;
  const int Bbytes = n.npad * Brow;
  img.assign(static_cast<size_t>(n.n_tiles) * n.KB * 2 * Bbytes, 0);
  const float wscale = std::ldexp(1.0f, -n.w_exp);
  auto wval = [&](int o, int k) -> float {
    if (o >= c.out_channels || k >= Kreal) return 0.0f;
    const int t = k / n.Csi, ch = k % n.Csi;
    if (ch >= c.in_channels) return 0.0f;
    const int kj = t / c.kernel_w, ki = t % c.kernel_w;
    return c.weights[((static_cast<size_t>(o) * c.in_channels + ch) * c.kernel_h + kj) * c.kernel_w + ki];
  };
  for (int nt = 0; nt < n.n_tiles; ++nt)
    for (int kb = 0; kb < n.KB; ++kb) {
      uint8_t* base = img.data() + (static_cast<size_t>(nt) * n.KB + kb) * 2 * Bbytes;
      for (int r = 0; r < n.npad; ++r) {
        if (f16) {
          // K-major SWIZZLE_64B: 64-B rows, 16-B chunk q at (q ^ ((r >> 1) & 3))
          for (int q = 0; q < 4; ++q)
            for (int j = 0; j < 8; ++j) {
              const float w = wval(nt * n.npad + r, kb * 32 + q * 8 + j) * wscale;  // exact (power of 2)
              const uint16_t hi = f16_rn(w);
              const uint16_t lo = f16_rn(w - f16_to_f32(hi));
              const size_t off = static_cast<size_t>(r) * 64 + ((q ^ ((r >> 1) & 3)) << 4) + j * 2;
              std::memcpy(base + off, &hi, 2);
              std::memcpy(base + Bbytes + off, &lo, 2);
            }
        } else {
          for (int q = 0; q < 8; ++q)
            for (int j = 0; j < 4; ++j) {
              const float w = wval(nt * n.npad + r, kb * 32 + q * 4 + j);
              const uint32_t hi = tf32_round(w);
              float hf;
              std::memcpy(&hf, &hi, 4);
              const uint32_t lo = tf32_round(w - hf);
              const size_t off = static_cast<size_t>(r) * 128 + ((q ^ (r & 7)) << 4) + j * 4;
              std::memcpy(base + off, &hi, 4);
              std::memcpy(base + Bbytes + off, &lo, 4);
            }
        }
      }
    }
  ktab.assign(static_cast<size_t>(n.KB) * 8 * 2, 0);
  for (int kb = 0; kb < n.KB; ++kb)
    for (int q = 0; q < 8; ++q) {
      const int k0 = kb * 32 + q * 4;
      const int t = k0 / n.Csi, c0 = k0 % n.Csi;
      if (t >= taps) {
        ktab[(kb * 8 + q) * 2] = 0x80000000u;
      } else {
        const int kj = t / c.kernel_w, ki = t % c.kernel_w;
        const long long off = (static_cast<long long>(kj) * n.d.Wi + ki) * n.Csi + c0;
        if (off > INT32_MAX) throw Error(CBG_ERR_UNSUPPORTED, "input row too large for 32-bit tap offsets");
        ktab[(kb * 8 + q) * 2 + 1] = static_cast<uint32_t>(off);
        ktab[(kb * 8 + q) * 2] = static_cast<uint32_t>(kj) | (static_cast<uint32_t>(ki) << 8) |
                           (static_cast<uint32_t>(c0) << 16);
      }
    }
  bias.assign(static_cast<size_t>(n.n_tiles) * n.npad, 0.0f);
  for (int o = 0; o < c.out_channels; ++o) bias[o] = c.bias[o];
}

// tcgen05 operand split: 3xFP16 with power-of-two scaling (default) or 3xTF32
// (CBG_GEMM_PREC=tf32); both fp32-accurate, DESIGN.md §3.3.
// A operand path of the fp16 split: loaded by the convert warps straight from
// global memory (2, default) or staged through shared memory by fetch warps
// (1, CBG_GEMM_DIRECT=0). Measured on the bench (64 streams, 4 overlapped
// stream groups): direct 50.0-50.6k frames/s, staged 48.7-49.2k, direct for
// N = 256 only 48.8-49.5k, although in an isolated launch the staged path is
// faster for N = 64 (L3 188 vs 204 us) and slower for N = 256 (L5 573 vs 552).
int gemm_prec(int npad) {
  const char* e = std::getenv("CBG_GEMM_PREC");
  if (e && std::strcmp(e, "tf32") == 0) return 0;
  const char* d = std::getenv("CBG_GEMM_DIRECT");
  if (d && std::strcmp(d, "0") == 0) return 1;
  (void)npad;
  return 2;
}

// Layers with at most this many output channels take the bit-exact CUDA-core
// path (conv_exact.cu); CBG_EXACT_MAX_COUT overrides it (0 = tcgen05 everywhere).
int exact_max_cout() {
  const char* e = std::getenv("CBG_EXACT_MAX_COUT");
  return e ? std::atoi(e) : 16;
}

// Compaction geometry of a node (kernels.hpp dilate_compact_tiling); Wp > 0: a fused pool's width.
DilateCompactArgs dc_geometry(int Hin, int Win, int Hout, int Wout, int kh, int kw, int stride, int pad, int S,
                              int Wp = 0) {
  if (Wout > 65536 || Win > 65536) throw Error(CBG_ERR_UNSUPPORTED, "map width > 65536 not supported");
  DilateCompactArgs g{};
  if (!dilate_compact_tiling(Hin, Win, Hout, Wout, kh, stride, Wp, &g.rows, &g.n_bands, &g.threads, &g.smem_bytes))
    throw Error(CBG_ERR_UNSUPPORTED, "compaction band exceeds 48 KB of shared memory");
  g.Hin = Hin, g.Win = Win, g.Hout = Hout, g.Wout = Wout;
  g.kh = kh, g.kw = kw, g.stride = stride, g.pad = pad;
  g.S = S;
  g.n_in = 1;
  return g;
}
size_t map_words_of(int H, int W) { return static_cast<size_t>(H) * ((W + 31) / 32); }
}  // namespace

Net::Net(Ctx* ctx, Topology topo, int n_streams) : ctx_(ctx), topo_(std::move(topo)), S_(n_streams) {
  if (S_ < 1 || S_ > 1024) throw_invalid("n_streams must be in [1, 1024]");
  build();
}

Net::~Net() {
  for (auto& g : graphs_) {
    cudaGraphExecDestroy(g.second.exec);
    cudaGraphDestroy(g.second.graph);
  }
  for (auto& e : ev_pool_) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    if (ev_copied_[b]) cudaEventDestroy(ev_copied_[b]);
    if (ev_consumed_[b]) cudaEventDestroy(ev_consumed_[b]);
  }
  if (copy_st_) {
    cudaStreamSynchronize(copy_st_);
    cudaStreamDestroy(copy_st_);
  }
  for (auto& e : ev_map_) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    if (ev_dstaged_[b]) cudaEventDestroy(ev_dstaged_[b]);
    if (ev_dpushed_[b]) {
      cudaEventSynchronize(ev_dpushed_[b]);
      cudaEventDestroy(ev_dpushed_[b]);
    }
  }
  for (auto& kv : delta_host_) cudaEventDestroy(kv.second.ev);
  for (int b = 0; b < 2; ++b) {
    if (ev_staged_[b]) cudaEventDestroy(ev_staged_[b]);
    if (ev_drained_[b]) {
      cudaEventSynchronize(ev_drained_[b]);
      cudaEventDestroy(ev_drained_[b]);
    }
  }
  if (side_st_) {
    cudaStreamSynchronize(side_st_);
    cudaStreamDestroy(side_st_);
  }
}

std::unique_ptr<Net> Net::clone() const {
  auto c = std::make_unique<Net>(ctx_, topo_, S_);
  CK(cudaStreamSynchronize(ctx_->stream));
  for (size_t i = 0; i < nodes_.size(); ++i) {
    const NodeRT& a = nodes_[i];
    NodeRT& b = c->nodes_[i];
    if (a.out.bytes) CK(cudaMemcpy(b.out.p, a.out.p, a.out.bytes, cudaMemcpyDeviceToDevice));
    if (a.state.bytes) CK(cudaMemcpy(b.state.p, a.state.p, a.state.bytes, cudaMemcpyDeviceToDevice));
    if (a.state8.bytes) CK(cudaMemcpy(b.state8.p, a.state8.p, a.state8.bytes, cudaMemcpyDeviceToDevice));
    if (a.split.bytes) {
      CK(cudaMemcpy(b.split.p, a.split.p, a.split.bytes, cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(b.split_e.p, a.split_e.p, a.split_e.bytes, cudaMemcpyDeviceToDevice));
    }
  }
  c->s8_valid_ = s8_valid_;
  c->s8_pending_ = s8_pending_;
  CK(cudaMemcpy(c->boot_req_.p, boot_req_.p, S_, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(c->amax_.p, amax_.p, amax_.bytes, cudaMemcpyDeviceToDevice));
  c->ext_amax_ = ext_amax_;
  c->host_taus_ = host_taus_;
  c->stream_taus_ = stream_taus_;
  CK(cudaMemcpy(c->taus_.p, taus_.p, taus_.bytes, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(c->rescan_req_.p, rescan_req_.p, rescan_req_.bytes, cudaMemcpyDeviceToDevice));
  c->set_dense(dense_);
  return c;
}

void Net::build() {
  CK(cudaSetDevice(ctx_->device));
  const int n = static_cast<int>(topo_.nodes.size());
  nodes_.resize(n);
  n_slots_ = 0;
  // count slots: external nodes' (uploaded by set_external) first, then the
  // per-frame atomic counters begin_frame zeroes
  for (int i = 0; i < n; ++i)
    if (topo_.nodes[i].kind == kExternal) nodes_[i].count_slot = n_slots_++;
  n_ext_slots_ = n_slots_;
  size_t clear_words = 0;  // arena of OR-written bitmaps
  std::vector<std::pair<int, size_t>> clear_off;
  for (int i = 0; i < n; ++i) {
    NodeRT& r = nodes_[i];
    r.d = topo_.nodes[i];
    const NodeDesc& d = r.d;
    r.Cs = round4(d.C);
    r.Csi = round4(d.Ci);
    const size_t HWo = static_cast<size_t>(d.H) * d.W;
    const size_t HWi = static_cast<size_t>(d.Hi) * d.Wi;
    r.out.alloc(static_cast<size_t>(S_) * HWo * r.Cs * sizeof(float));
    const bool reuse = d.kind == CBG_LAYER_CONV && d.policy == CBG_POLICY_REUSE1X1;
    if (reuse) {
      const NodeRT& prod = nodes_[d.inputs[0]];
      r.outmap = prod.outmap;
      r.idx = prod.idx;
      r.count_slot = prod.count_slot;
    } else {
      r.outmap_own.alloc(static_cast<size_t>(S_) * map_words_of(d.H, d.W) * 4);
      r.idx_own.alloc(static_cast<size_t>(S_) * HWo * sizeof(int32_t));
      r.outmap = r.outmap_own.as<uint32_t>();
      r.idx = r.idx_own.as<int32_t>();
      if (d.kind != kExternal) r.count_slot = n_slots_++;
    }
    if (d.kind == kExternal) continue;
    if (d.kind == CBG_LAYER_CONV) {
      const ConvDesc& c = d.conv;
      if (c.kernel_h > 255 || c.kernel_w > 255) throw Error(CBG_ERR_UNSUPPORTED, "kernel dims > 255");
      const int Co4 = r.Cs;
      r.npad = Co4 <= 16 ? 16 : Co4 <= 32 ? 32 : Co4 <= 64 ? 64 : Co4 <= 128 ? 128 : 256;
      r.n_tiles = (Co4 + r.npad - 1) / r.npad;
      const int K = c.kernel_h * c.kernel_w * r.Csi;
      r.KB = (K + 31) / 32;
      const int Kref = c.in_channels * c.kernel_h * c.kernel_w;
      r.exact = c.out_channels <= exact_max_cout() && conv_exact_supported(c.kernel_w) && conv_exact_smem_bytes(c.out_channels, Kref) <= 192 * 1024;
      std::vector<float> bias;
      if (r.exact) {
        r.wraw.alloc(c.weights.size() * sizeof(float));
        CK(cudaMemcpy(r.wraw.p, c.weights.data(), c.weights.size() * sizeof(float), cudaMemcpyHostToDevice));
        bias.assign(c.bias.begin(), c.bias.end());
      } else {
        if (r.KB > 512) throw Error(CBG_ERR_UNSUPPORTED, "Cin*kh*kw too large for the GEMM kernel (K > 16384)");
        if (r.Csi >= 32768) throw Error(CBG_ERR_UNSUPPORTED, "too many input channels");
        r.prec = gemm_prec(r.npad);
        {
          const char* te = std::getenv("CBG_TMA_1X1");
          r.tma_a = te && std::atoi(te) != 0 && c.kernel_h == 1 && c.kernel_w == 1 && c.stride == 1 &&
                    c.padding == 0 && r.prec == 2;
          if (r.tma_a) r.prec = 1;  // staged A path, rows by TMA
        }
        constexpr int kSmemMax = 232448;  // 227 KB opt-in per CTA
        if (conv_gemm_smem_bytes(r.npad, r.KB, S_, r.prec, r.n_tiles) > kSmemMax) r.prec = 0;  // fewer stages (tf32)
        if (conv_gemm_smem_bytes(r.npad, r.KB, S_, r.prec, r.n_tiles) > kSmemMax)
          throw Error(CBG_ERR_UNSUPPORTED, "conv layer too large for the GEMM kernel's shared memory (K or streams)");
        r.w_exp = r.prec != 0 ? weight_exp(c.weights) : 0;
        std::vector<uint8_t> img;
        std::vector<uint32_t> ktab;
        build_weight_image(r, img, ktab, bias);
        r.wimg.alloc(img.size());
        CK(cudaMemcpy(r.wimg.p, img.data(), img.size(), cudaMemcpyHostToDevice));
        r.ktab.alloc(ktab.size() * 4);
        CK(cudaMemcpy(r.ktab.p, ktab.data(), ktab.size() * 4, cudaMemcpyHostToDevice));
      }
      r.bias.alloc(bias.size() * 4);
      CK(cudaMemcpy(r.bias.p, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
      if (d.policy == CBG_POLICY_DETECT) {
        r.state_chw = r.exact && d.inputs[0] < 0;
        r.state.alloc(static_cast<size_t>(S_) * HWi * (r.state_chw ? d.Ci : r.Csi) * sizeof(float));
        if (r.state_chw && d.Ci == 3 && HWi % 4 == 0) r.state8.alloc(static_cast<size_t>(S_) * HWi * 3 + 16);
        r.det_slot = n_slots_++;
        r.inmap_words = static_cast<size_t>(S_) * map_words_of(d.Hi, d.Wi);
        r.inmap_plain = d.inputs[0] < 0 && detect_frame_plain_map(d.Ci, r.Csi, d.Wi, r.state_chw ? 1 : 0);
        clear_off.push_back({i, clear_words});
        clear_words += (r.inmap_words + 3) & ~static_cast<size_t>(3);  // 16-B aligned
        // the direct 3xFP16 GEMM of a k x k layer (k > 1) gathers every input value
        // k^2 times: its detect keeps the state pre-split, once per changed pixel
        const char* ps_env = std::getenv("CBG_PRESPLIT");  // read per build: A/B in one process
        const bool presplit = !(ps_env && std::atoi(ps_env) == 0);
        if (presplit && !r.exact && r.prec == 2 && d.inputs[0] >= 0 && nodes_[d.inputs[0]].d.kind != kExternal &&
            c.kernel_h * c.kernel_w > 1) {
          r.split.alloc(r.state.bytes);
          r.split_e.alloc(2 * static_cast<size_t>(S_) * sizeof(int32_t));
          CK(cudaMemset(r.split_e.p, 0x7f, r.split_e.bytes));  // no exponent yet: the first frame splits all
          CK(cudaStreamSynchronize(nullptr));
        }
      }
      if (!reuse && (d.policy == CBG_POLICY_DETECT || d.policy == CBG_POLICY_PROPAGATE))
        r.dc = dc_geometry(d.Hi, d.Wi, d.H, d.W, c.kernel_h, c.kernel_w, c.stride, c.padding, S_);
      // worst-case map buffers (record_worst_case, layers.cpp:108-117)
      if (d.inputs[0] >= 0) {
        r.dc_wc = dc_geometry(d.Hi, d.Wi, d.H, d.W, c.kernel_h, c.kernel_w, c.stride, c.padding, S_);
        r.wc_map.alloc(static_cast<size_t>(S_) * map_words_of(d.H, d.W) * 4);
        r.wc_idx.alloc(static_cast<size_t>(S_) * HWo * sizeof(int32_t));
      }
      r.wc_slot = n_slots_++;
    } else if (d.kind == CBG_LAYER_POOL) {
      // a 2x2 / stride-2 pool over a node that runs its own compaction gets its
      // map and list from that compaction (one launch fewer, no map re-read)
      NodeRT& p = nodes_[d.inputs[0]];
      const bool host = p.d.kind != kExternal && p.dc.n_bands > 0 && p.pool_child < 0 && p.fused_into < 0 &&
                        !(p.d.kind == CBG_LAYER_CONV && p.d.policy == CBG_POLICY_REUSE1X1);
      const char* fe = std::getenv("CBG_FUSE_POOL");
      if (host && d.pool_size == 2 && d.pool_stride == 2 && !(fe && std::atoi(fe) == 0)) {
        DilateCompactArgs g = p.dc;
        DilateCompactArgs f = dc_geometry(g.Hin, g.Win, g.Hout, g.Wout, g.kh, g.kw, g.stride, g.pad, S_, d.W);
        p.dc = f;
        p.pool_child = i;
        r.fused_into = d.inputs[0];
      } else {
        r.dc = dc_geometry(d.Hi, d.Wi, d.H, d.W, d.pool_size, d.pool_size, d.pool_stride, 0, S_);
      }
    } else if (d.kind == CBG_LAYER_UPSAMPLE) {
      r.dc = dc_geometry(d.Hi, d.Wi, d.H, d.W, 1, 1, 1, 0, S_);
      r.dc.up = d.up;
    } else {  // joins: OR of the parents' maps, 1x1 identity window
      r.dc = dc_geometry(d.H, d.W, d.H, d.W, 1, 1, 1, 0, S_);
    }
  }
  if (clear_words) {
    clear_.alloc(clear_words * 4);
    for (auto& [i, off] : clear_off) nodes_[i].inmap = clear_.as<uint32_t>() + off;
  }
  frame_.alloc(static_cast<size_t>(S_) * topo_.C * topo_.H * topo_.W * sizeof(float));
  frame_slot_.alloc(sizeof(void*));
  {
    const float* p = frame_.as<float>();
    CK(cudaMemcpy(frame_slot_.p, &p, sizeof(p), cudaMemcpyHostToDevice));
  }
  if (const char* e = std::getenv("CBG_SIDE_DILCOMP")) side_dc_ = std::atoi(e) != 0;
  CK(cudaStreamCreateWithFlags(&side_st_, cudaStreamNonBlocking));
  ev_map_.resize(nodes_.size());
  for (auto& e : ev_map_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  frame_ctr_.alloc(4);
  boot_req_.alloc(S_);
  // a network bootstraps on its first frame (network.cpp:318-321); a standalone
  // layer does not: only force_full_update makes it a full update (layers.cpp:64-71)
  if (n == 0 || nodes_[0].d.kind != kExternal) CK(cudaMemset(boot_req_.p, 1, S_));
  CK(cudaStreamSynchronize(nullptr));
  s8_valid_.assign(S_, 0);
  s8_pending_.assign(S_, 1);
  boot_now_.alloc(S_);
  dense_flag_.alloc(1);
  rescan_req_.alloc(std::max(1, n));
  rescan_now_.alloc(std::max(1, n));
  taus_.alloc(static_cast<size_t>(std::max(1, n)) * S_ * sizeof(float));
  host_taus_.assign(n, 0.0f);
  stream_taus_.assign(static_cast<size_t>(n) * S_, 0.0f);
  for (int i = 0; i < n; ++i) {
    host_taus_[i] = nodes_[i].d.tau;
    for (int k = 0; k < S_; ++k) stream_taus_[static_cast<size_t>(i) * S_ + k] = nodes_[i].d.tau;
  }
  if (n) CK(cudaMemcpy(taus_.p, stream_taus_.data(), stream_taus_.size() * sizeof(float), cudaMemcpyHostToDevice));
  // [S][cnt_stride_]: each stream's counters in their own cache lines, so the
  // per-warp / per-CTA atomics of different streams never share a line
  cnt_stride_ = (std::max(1, n_slots_) + 31) / 32 * 32;
  counts_.alloc(static_cast<size_t>(cnt_stride_) * S_ * sizeof(int32_t));
  amax_.alloc(static_cast<size_t>(n + 1) * S_ * sizeof(float));
  ext_amax_.assign(S_, 0.0f);
}

int Net::amax_origin(int node) const {
  while (node >= 0 && (nodes_[node].d.kind == CBG_LAYER_POOL || nodes_[node].d.kind == CBG_LAYER_UPSAMPLE))
    node = nodes_[node].d.inputs[0];
  return node;  // -1 = network input
}

int Net::launch_count(unsigned flags) const {
  int k = 1;  // begin_frame
  for (const NodeRT& r : nodes_) {
    const NodeDesc& d = r.d;
    if (d.kind == kExternal) continue;
    if (d.kind == CBG_LAYER_CONV) {
      k += (d.policy == CBG_POLICY_DETECT) + (d.policy != CBG_POLICY_REUSE1X1) + 1;
      if ((flags & CBG_FWD_RECORD_WORST_CASE) && d.inputs[0] >= 0) k += 1;
    } else {
      k += r.fused_into >= 0 ? 1 : 2;
    }
  }
  return k;
}

void Net::enqueue_frame(unsigned flags, bool u8, bool bcast, int slot8, bool s8) {
  cudaStream_t st = ctx_->stream;
  int32_t* counts = counts_.as<int32_t>();
  const uint32_t* frame = frame_ctr_.as<uint32_t>();
  const uint8_t* boot = boot_now_.as<uint8_t>();
  const int n = static_cast<int>(nodes_.size());
  {
    const bool ext_in = n > 0 && nodes_[0].d.kind == kExternal;
    const void** in_slot = ext_in ? nullptr
                           : u8  ? (slot8 == 2 ? reinterpret_cast<const void**>(frame8_slot_.as<const uint8_t*>() + 2)
                                               : nullptr)
                                 : reinterpret_cast<const void**>(frame_slot_.p);
    BeginFrameArgs b{frame_ctr_.as<uint32_t>(), boot_now_.as<uint8_t>(), boot_req_.as<uint8_t>(),
                     dense_flag_.as<uint8_t>(), rescan_now_.as<uint8_t>(), rescan_req_.as<uint8_t>(),
                     counts, cnt_stride_ * S_, cnt_stride_, n_ext_slots_,
                     clear_.as<uint4>(), static_cast<long long>(clear_.bytes / 16), S_, n,
                     in_slot ? in_ptr_ : nullptr, in_slot};
    timed("frame.begin", [&] { launch_begin_frame(b, st); });
  }
  // node whose compaction wrote node k's map (Reuse1x1 nodes alias their producer's)
  auto map_owner = [&](int k) {
    while (nodes_[k].d.kind == CBG_LAYER_CONV && nodes_[k].d.policy == CBG_POLICY_REUSE1X1) k = nodes_[k].d.inputs[0];
    return k;
  };
  // the compaction of node k (its geometry, maps and list), with its fused pool's outputs
  auto compaction = [&](int k, const uint32_t* const* in, int n_in) {
    const NodeRT& r = nodes_[k];
    DilateCompactArgs dc = r.dc;
    for (int q = 0; q < n_in; ++q) dc.in_map[q] = in[q];
    dc.n_in = n_in;
    dc.out_map = r.outmap;
    dc.idx = r.idx;
    dc.count = counts + r.count_slot;
    dc.cnt_stride = cnt_stride_;
    dc.boot = boot;
    if (r.pool_child >= 0) {
      const NodeRT& p = nodes_[r.pool_child];
      dc.pool_map = p.outmap;
      dc.pool_idx = p.idx;
      dc.pool_count = counts + p.count_slot;
      dc.Hp = p.d.H, dc.Wp = p.d.W;
    }
    return dc;
  };
  auto done_map = [&](int k, cudaStream_t on) {
    CK(cudaEventRecord(ev_map_[k], on));
    if (nodes_[k].pool_child >= 0) CK(cudaEventRecord(ev_map_[nodes_[k].pool_child], on));
  };
  // compaction of node k from its producers' maps: on the side stream once
  // those maps exist (their GEMMs may still run), then joined back
  auto map_compaction = [&](int k, const DilateCompactArgs& dc) {
    const NodeDesc& dk = nodes_[k].d;
    bool side = side_dc_ && !timing_;  // per-kernel timing keeps every kernel on the ctx stream (serial attribution)
    for (int in : dk.inputs) side = side && nodes_[map_owner(in)].d.kind != kExternal;
    if (!side) {
      timed(dk.name + ".dilcomp", [&] { launch_dilate_compact(dc, st); });
      done_map(k, st);
      return;
    }
    for (int in : dk.inputs) CK(cudaStreamWaitEvent(side_st_, ev_map_[map_owner(in)], 0));
    timed(dk.name + ".dilcomp", [&] { launch_dilate_compact(dc, side_st_); }, side_st_);
    done_map(k, side_st_);
    CK(cudaStreamWaitEvent(st, ev_map_[k], 0));
  };
  for (int i = 0; i < n; ++i) {
    NodeRT& r = nodes_[i];
    const NodeDesc& d = r.d;
    if (d.kind == kExternal) continue;
    const int src = d.inputs[0];
    const NodeRT* prod = src >= 0 ? &nodes_[src] : nullptr;
    if (d.kind == CBG_LAYER_CONV) {
      const ConvDesc& c = d.conv;
      const float* column_src = prod ? prod->out.as<float>() : nullptr;
      if (d.policy == CBG_POLICY_DETECT) {
        int32_t* det = counts + r.det_slot;
        if (!prod) {
          DetectFrameArgs a{};
          a.x_slot = frame_slot_.as<const float*>();
          a.state = r.state.as<float>();
          a.map = r.inmap;
          a.map_plain = r.inmap_plain ? 1 : 0;
          a.det_count = det;
          a.cnt_stride = cnt_stride_;
          a.boot = boot;
          a.C = d.Ci, a.Cs = r.Csi, a.H = d.Hi, a.W = d.Wi, a.S = S_;
          a.tau = taus_.as<float>() + static_cast<size_t>(i) * S_;
          a.closed_loop = topo_.mode == CBG_MODE_CLOSEDLOOP;
          a.state_chw = r.state_chw;
          a.amax = amax_entry(-1);
          a.x8_slot = u8 ? frame8_slot_.as<const uint8_t*>() + slot8 : nullptr;
          a.x_sstride = bcast ? 0LL : static_cast<long long>(d.Ci) * d.Hi * d.Wi;
          a.state8 = u8 ? r.state8.as<uint8_t>() : nullptr;
          a.use_state8 = (u8 && s8) ? 1 : 0;
          timed(d.name + ".detect", [&] { launch_detect_frame(a, st); });
        } else {
          const bool ext = prod->d.kind == kExternal;  // standalone layer: arbitrary x, dense detect
          DetectListArgs a{prod->out.as<float>(), r.state.as<float>(), r.inmap, det,
                           ext ? nullptr : prod->idx, counts + prod->count_slot, frame, boot,
                           rescan_now_.as<uint8_t>() + i, r.Csi, d.Hi, d.Wi, S_,
                           taus_.as<float>() + static_cast<size_t>(i) * S_,
                           topo_.mode == CBG_MODE_CLOSEDLOOP, cnt_stride_,
                           r.split.bytes ? r.split.as<uint32_t>() : nullptr, r.split_e.as<int32_t>(),
                           amax_entry(amax_origin(src))};
          timed(d.name + ".detect", [&] { launch_detect_list(a, st); });
        }
        // ClosedLoop reads the state; FeedForward's state equals x after detection.
        column_src = r.state.as<float>();
        const uint32_t* in[1] = {r.inmap};
        const DilateCompactArgs dc = compaction(i, in, 1);
        timed(d.name + ".dilcomp", [&] { launch_dilate_compact(dc, st); });
        done_map(i, st);
      } else if (d.policy == CBG_POLICY_PROPAGATE) {
        const uint32_t* in[1] = {prod->outmap};
        map_compaction(i, compaction(i, in, 1));
      }
      if ((flags & CBG_FWD_RECORD_WORST_CASE) && prod) {
        DilateCompactArgs dc = r.dc_wc;
        dc.in_map[0] = prod->outmap;
        dc.n_in = 1;
        dc.out_map = r.wc_map.as<uint32_t>();
        dc.idx = r.wc_idx.as<int32_t>();
        dc.count = counts + r.wc_slot;
        dc.cnt_stride = cnt_stride_;
        dc.boot = boot;
        timed(d.name + ".worstcase", [&] { launch_dilate_compact(dc, st); });
      }
      if (r.exact) {
        ConvExactArgs x{};
        x.src = column_src;
        if (r.state_chw) {
          x.src_sstride = static_cast<long long>(d.Hi) * d.Wi * d.Ci;
          x.cstride = static_cast<long long>(d.Hi) * d.Wi;
          x.pstride = 1;
        } else {
          x.src_sstride = static_cast<long long>(d.Hi) * d.Wi * r.Csi;
          x.cstride = 1;
          x.pstride = r.Csi;
        }
        x.out = r.out.as<float>();
        x.idx = r.idx;
        x.count = counts + r.count_slot;
        x.cnt_stride = cnt_stride_;
        x.w = r.wraw.as<float>();
        x.bias = r.bias.as<float>();
        x.Cin = c.in_channels, x.Cout = c.out_channels, x.Co4 = r.Cs;
        x.kh = c.kernel_h, x.kw = c.kernel_w, x.stride = c.stride, x.pad = c.padding;
        x.Hin = d.Hi, x.Win = d.Wi, x.Hout = d.H, x.Wout = d.W;
        x.relu = d.relu;
        x.slope = d.slope;
        x.S = S_;
        // the CUDA-core conv keeps every SM (measured: 60.4k vs 59.3k frames/s with
        // the GEMMs' share); CBG_EXACT_SMS=-1 gives it the share, n > 0 n SMs
        {
          static const int ectas = std::getenv("CBG_EXACT_SMS") ? std::atoi(std::getenv("CBG_EXACT_SMS")) : 0;
          x.sm_count = ectas == 0 ? ctx_->sm_count : ectas > 0 ? std::min(ectas, ctx_->sm_count) : ctx_->persistent();
        }
        x.amax_out = amax_entry(i);
        timed(d.name + ".gemm", [&] { launch_conv_exact(x, st); });
        continue;
      }
      ConvGemmArgs g{};
      g.src = column_src;
      if (r.split.bytes) {  // the detect's pre-split copy of the same state
        g.src = static_cast<const float*>(r.split.p);
        g.src_presplit = 1;
      }
      g.out = r.out.as<float>();
      g.idx = r.idx;
      g.count = counts + r.count_slot;
      g.cnt_stride = cnt_stride_;
      g.wimg = r.wimg.as<uint8_t>();
      g.ktab = r.ktab.as<uint32_t>();
      g.bias = r.bias.as<float>();
      g.Cs = r.Csi, g.Hin = d.Hi, g.Win = d.Wi, g.Hout = d.H, g.Wout = d.W, g.Co4 = r.Cs;
      g.stride = c.stride, g.pad = c.padding;
      g.kh = c.kernel_h, g.kw = c.kernel_w;
      g.KB = r.KB, g.npad = r.npad, g.n_tiles = r.n_tiles;
      if (r.tma_a) {  // TMA gather4 map of the column source [S*Hi*Wi][Csi] fp32 (encoded once per source)
        if (r.tmap_src != g.src) {
          using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
          static EncodeFn encode = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
            return reinterpret_cast<EncodeFn>(fn);
          }();
          const cuuint64_t dims[2] = {static_cast<cuuint64_t>(r.Csi), static_cast<cuuint64_t>(S_) * d.Hi * d.Wi};
          const cuuint64_t strides[1] = {static_cast<cuuint64_t>(r.Csi) * 4};
          const cuuint32_t box[2] = {32, 1};
          const cuuint32_t estr[2] = {1, 1};
          if (encode(&r.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(g.src), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            throw Error(CBG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
          r.tmap_src = g.src;
        }
        g.tmap = r.tmap;
        g.use_tma = 1;
      }
      g.relu = d.relu;
      g.slope = d.slope;
      g.S = S_;
      g.grid = ctx_->persistent();  // (the share for L5 alone: 58.8k vs 60.2k frames/s with it for every GEMM)
      g.prec = r.prec;
      g.w_exp = r.w_exp;
      g.amax_in = amax_entry(amax_origin(src));  // state / producer output values come from here
      g.amax_out = amax_entry(i);
      timed(d.name + ".gemm", [&] { launch_conv_gemm(g, st); });
    } else if (d.kind == CBG_LAYER_POOL) {
      if (r.fused_into < 0) {
        const uint32_t* in[1] = {prod->outmap};
        map_compaction(i, compaction(i, in, 1));
      }
      PoolArgs pa{prod->out.as<float>(), r.out.as<float>(), r.idx, counts + r.count_slot, r.Cs, d.Hi, d.Wi,
                  d.H, d.W, d.pool_size, d.pool_stride, S_, cnt_stride_};
      timed(d.name + ".pool", [&] { launch_pool(pa, st); });
    } else if (d.kind == CBG_LAYER_UPSAMPLE) {
      const uint32_t* in[1] = {prod->outmap};
      map_compaction(i, compaction(i, in, 1));
      PoolArgs pa{prod->out.as<float>(), r.out.as<float>(), r.idx, counts + r.count_slot, r.Cs, d.Hi, d.Wi,
                  d.H, d.W, 0, d.up, S_, cnt_stride_};
      timed(d.name + ".upsample", [&] { launch_upsample(pa, st); });
    } else {  // Add / Concat
      const uint32_t* in[4] = {};
      for (size_t k = 0; k < d.inputs.size(); ++k) in[k] = nodes_[d.inputs[k]].outmap;
      map_compaction(i, compaction(i, in, static_cast<int>(d.inputs.size())));
      JoinArgs ja{};
      for (size_t k = 0; k < d.inputs.size(); ++k) {
        const NodeRT& p = nodes_[d.inputs[k]];
        ja.in[k] = p.out.as<float>();
        ja.in_cs[k] = p.Cs;
        ja.in_c[k] = p.d.C;
      }
      ja.n_in = static_cast<int>(d.inputs.size());
      ja.is_add = d.kind == CBG_LAYER_ADD;
      ja.out = r.out.as<float>();
      ja.Cs_out = r.Cs;
      ja.idx = r.idx;
      ja.count = counts + r.count_slot;
      ja.cnt_stride = cnt_stride_;
      ja.HW = d.H * d.W;
      ja.S = S_;
      ja.amax_out = amax_entry(i);
      timed(d.name + ".join", [&] { launch_join(ja, st); });
    }
  }
}

void Net::forward(const float* frames, unsigned flags) {
  cudaStream_t st = ctx_->stream;
  CK(cudaSetDevice(ctx_->device));
  const bool ext = !nodes_.empty() && nodes_[0].d.kind == kExternal;
  if (!ext) {
    if (frames == nullptr) throw_invalid("forward_frame: null frame");
    // zero-copy for device inputs: the ingest kernel reads through a device
    // pointer slot that begin_frame fills (a kernel-node parameter of the
    // captured graph, set per launch), so one graph serves any input buffer
    in_ptr_ = (flags & CBG_FWD_INPUT_ON_DEVICE) ? frames : frame_.as<float>();
    if (!(flags & CBG_FWD_INPUT_ON_DEVICE))
      CK(cudaMemcpyAsync(frame_.p, frames, (flags & CBG_FWD_BROADCAST_INPUT) ? frame_.bytes / S_ : frame_.bytes,
                         cudaMemcpyHostToDevice, st));
  }
  run_frame(flags, (flags & CBG_FWD_RECORD_WORST_CASE) | ((flags & CBG_FWD_BROADCAST_INPUT) ? (1u << 30) : 0u));
  // fp32 values in the state: the 8-bit shadow is stale until a full update
  // goes through the 8-bit ingest (a boot here consumed the pending requests)
  std::fill(s8_valid_.begin(), s8_valid_.end(), 0);
  std::fill(s8_pending_.begin(), s8_pending_.end(), 0);
}

void Net::forward_u8(const uint8_t* frames, unsigned flags) {
  cudaStream_t st = ctx_->stream;
  CK(cudaSetDevice(ctx_->device));
  if (!nodes_.empty() && nodes_[0].d.kind == kExternal) throw_invalid("forward_u8: standalone layers take fp32 input");
  if (frames == nullptr) throw_invalid("forward_u8: null frame");
  if (topo_.C > 4) throw Error(CBG_ERR_UNSUPPORTED, "8-bit ingest supports at most 4 input channels (PNM: 1 or 3)");
  bool first_detect = false;
  for (const NodeRT& r : nodes_)
    if (r.d.kind == CBG_LAYER_CONV && r.d.inputs[0] < 0 && r.d.policy == CBG_POLICY_DETECT) first_detect = true;
  if (!first_detect) throw Error(CBG_ERR_UNSUPPORTED, "8-bit ingest needs a detect-policy first layer");
  const size_t fbytes = static_cast<size_t>(S_) * topo_.H * topo_.W * topo_.C;
  if (!frame8_.bytes) {
    frame8_.alloc(2 * fbytes);
    frame8_slot_.alloc(3 * sizeof(void*));
    const uint8_t* v[3] = {frame8_.as<uint8_t>(), frame8_.as<uint8_t>() + fbytes, nullptr};
    CK(cudaMemcpy(frame8_slot_.p, v, sizeof(v), cudaMemcpyHostToDevice));
    CK(cudaStreamCreateWithFlags(&copy_st_, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&ev_copied_[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_consumed_[b], cudaEventDisableTiming));
    }
  }
  if (flags & CBG_FWD_FORCE_FULL) std::fill(s8_pending_.begin(), s8_pending_.end(), 1);
  bool s8 = true;  // every first layer keeps a valid 8-bit shadow for every stream
  for (const NodeRT& r : nodes_)
    if (r.d.kind == CBG_LAYER_CONV && r.d.inputs[0] < 0 && r.d.policy == CBG_POLICY_DETECT)
      s8 = s8 && r.state8.bytes != 0;
  for (uint8_t v : s8_valid_) s8 = s8 && v;
  const unsigned key = (flags & CBG_FWD_RECORD_WORST_CASE) | (1u << 31) | (s8 ? (1u << 27) : 0u);
  // after the frame: streams that took a full update hold a valid shadow
  auto s8_after = [&] {
    const bool all = dense_ || topo_.mode != CBG_MODE_CLOSEDLOOP;
    for (size_t k = 0; k < s8_valid_.size(); ++k) {
      if (all || s8_pending_[k]) s8_valid_[k] = 1;
      s8_pending_[k] = 0;
    }
  };
  if (flags & CBG_FWD_INPUT_ON_DEVICE) {
    in_ptr_ = frames;  // into pointer slot 2 by begin_frame (no copy of the slot)
    run_frame(flags, key | (2u << 28));
    s8_after();
    return;
  }
  // host frames: H2D into buffer b on the copy stream once the frame that last
  // read b (two calls ago) is done, so the copy overlaps the previous frame
  const int b = u8_buf_;
  u8_buf_ ^= 1;
  CK(cudaStreamWaitEvent(copy_st_, ev_consumed_[b], 0));
  CK(cudaMemcpyAsync(frame8_.as<uint8_t>() + b * fbytes, frames, fbytes, cudaMemcpyHostToDevice, copy_st_));
  CK(cudaEventRecord(ev_copied_[b], copy_st_));
  CK(cudaStreamWaitEvent(st, ev_copied_[b], 0));
  run_frame(flags, key | (static_cast<unsigned>(b) << 28));
  s8_after();
  CK(cudaEventRecord(ev_consumed_[b], st));
}

// One frame step: bookkeeping, then the captured graph for this flag set
// (graph_key bit 31 = 8-bit ingest).
void Net::run_frame(unsigned flags, unsigned graph_key) {
  cudaStream_t st = ctx_->stream;
  if (flags & CBG_FWD_FORCE_FULL) CK(cudaMemsetAsync(boot_req_.p, 1, S_, st));
  ++host_frame_;
  const unsigned gflags = flags & CBG_FWD_RECORD_WORST_CASE;
  const bool u8 = (graph_key >> 31) != 0;
  const bool bcast = ((graph_key >> 30) & 1u) != 0;
  const int slot8 = static_cast<int>((graph_key >> 28) & 3u);
  const bool s8 = ((graph_key >> 27) & 1u) != 0;
  last_flags_ = flags;
  last_launches_ = launch_count(gflags);
  if (timing_) {
    enqueue_frame(gflags, u8, bcast, slot8, s8);
    CK(cudaStreamSynchronize(st));
    size_t k = 0;
    for (auto& p : pending_) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
      auto& acc = times_[p.first];
      acc.first += ms;
      acc.second += 1;
      ev_pool_[k++] = p.second.first;
      ev_pool_[k++] = p.second.second;
    }
    pending_.clear();
    ++timed_frames_;
    CK(cudaGetLastError());
    return;
  }
  auto it = graphs_.find(graph_key);
  if (it == graphs_.end()) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_frame(gflags, u8, bcast, slot8, s8);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      throw;
    }
    CK(cudaStreamEndCapture(st, &g));
    GraphRec rec;
    rec.graph = g;
    size_t n_roots = 0;
    CK(cudaGraphGetRootNodes(g, nullptr, &n_roots));
    std::vector<cudaGraphNode_t> roots(n_roots);
    if (n_roots) CK(cudaGraphGetRootNodes(g, roots.data(), &n_roots));
    for (cudaGraphNode_t nd : roots) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams p{};
      CK(cudaGraphKernelNodeGetParams(nd, &p));
      if (p.func != begin_frame_fn()) continue;
      rec.begin = nd;
      rec.begin_params = p;
      rec.begin_args = *static_cast<const BeginFrameArgs*>(p.kernelParams[0]);
    }
    if (!rec.begin) throw Error(CBG_ERR_CUDA, "captured frame graph has no begin_frame root");
    CK(cudaGraphInstantiate(&rec.exec, g, 0));
    it = graphs_.emplace(graph_key, rec).first;
  }
  GraphRec& rec = it->second;
  if (rec.begin_args.in_slot && rec.begin_args.in_ptr != in_ptr_) {  // this frame's input buffer
    rec.begin_args.in_ptr = in_ptr_;
    void* kp[1] = {&rec.begin_args};
    cudaKernelNodeParams p = rec.begin_params;
    p.kernelParams = kp;
    p.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(rec.exec, rec.begin, &p));
  }
  CK(cudaGraphLaunch(rec.exec, st));
  CK(cudaGetLastError());
}

template <class F>
void Net::timed(const std::string& label, F&& launch, cudaStream_t on) {
  if (dry_) {
    dry_labels_.push_back(label);
    return;
  }
  if (!timing_) {
    launch();
    return;
  }
  if (!on) on = ctx_->stream;
  const size_t need = 2 * (pending_.size() + 1);
  while (ev_pool_.size() < need) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  cudaEvent_t a = ev_pool_[need - 2], b = ev_pool_[need - 1];
  CK(cudaEventRecord(a, on));
  launch();
  CK(cudaEventRecord(b, on));
  pending_.push_back({label, {a, b}});
}

std::vector<std::string> Net::kernel_labels(unsigned flags) {
  dry_ = true;
  dry_labels_.clear();
  try {
    enqueue_frame(flags & CBG_FWD_RECORD_WORST_CASE);
  } catch (...) {
    dry_ = false;
    throw;
  }
  dry_ = false;
  CK(cudaStreamSynchronize(ctx_->stream));  // (event records / waits only)
  CK(cudaStreamSynchronize(side_st_));
  return std::move(dry_labels_);
}

void Net::set_timing(bool on) {
  timing_ = on;
  times_.clear();
  timed_frames_ = 0;
}

std::string Net::timing_report() const {
  std::string js = "{\"frames\": " + std::to_string(timed_frames_) + ", \"kernels\": {";
  bool first = true;
  for (const auto& kv : times_) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s\"%s\": [%.6f, %lld]", first ? "" : ", ", kv.first.c_str(), kv.second.first,
                  kv.second.second);
    js += buf;
    first = false;
  }
  return js + "}}";
}

void Net::copy_counts_async(int32_t* host_dst) {
  CK(cudaMemcpyAsync(host_dst, counts_.p, counts_.bytes,
                     cudaMemcpyDeviceToHost, ctx_->stream));
}

void Net::copy_output_async(int node, void* host_dst) {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size())) throw_invalid("copy_output_async: bad node");
  const NodeRT& r = nodes_[node];
  CK(cudaMemcpyAsync(host_dst, r.out.p, r.out.bytes, cudaMemcpyDeviceToHost, ctx_->stream));
}

void Net::copy_output_detached(int node, void* host_dst) {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size())) throw_invalid("copy_output_detached: bad node");
  const NodeRT& r = nodes_[node];
  cudaStream_t st = ctx_->stream;
  if (!ev_staged_[0])
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&ev_staged_[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_drained_[b], cudaEventDisableTiming));
    }
  const int b = out_buf_;
  out_buf_ ^= 1;
  if (out_stage_[b].bytes < r.out.bytes) {
    CK(cudaEventSynchronize(ev_drained_[b]));
    out_stage_[b].alloc(r.out.bytes);
  }
  // staging b is free once its previous D2H (two calls ago) has drained
  CK(cudaStreamWaitEvent(st, ev_drained_[b], 0));
  CK(cudaMemcpyAsync(out_stage_[b].p, r.out.p, r.out.bytes, cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(ev_staged_[b], st));
  CK(cudaStreamWaitEvent(ctx_->d2h, ev_staged_[b], 0));
  CK(cudaMemcpyAsync(host_dst, out_stage_[b].p, r.out.bytes, cudaMemcpyDeviceToHost, ctx_->d2h));
  CK(cudaEventRecord(ev_drained_[b], ctx_->d2h));
}

size_t Net::output_delta_bytes(int node) const {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size())) throw_invalid("output_delta_bytes: bad node");
  const NodeRT& r = nodes_[node];
  const long long HW = static_cast<long long>(r.d.H) * r.d.W;
  return delta_header_bytes(S_) + static_cast<size_t>(S_) * delta_stream_bytes(HW, r.Cs);
}

void Net::copy_output_delta(int node, void* host_buf) {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size())) throw_invalid("copy_output_delta: bad node");
  const NodeRT& r = nodes_[node];
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, host_buf, 0) != cudaSuccess || dptr == nullptr) {
    cudaGetLastError();
    throw_invalid("copy_output_delta: host buffer is not pinned, mapped host memory");
  }
  cudaStream_t st = ctx_->stream;
  const size_t cap = output_delta_bytes(node);
  if (!ev_dstaged_[0])
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&ev_dstaged_[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_dpushed_[b], cudaEventDisableTiming));
    }
  const int b = delta_buf_;
  delta_buf_ ^= 1;
  if (delta_stage_[b].bytes < cap) {
    CK(cudaEventSynchronize(ev_dpushed_[b]));
    delta_stage_[b].alloc(cap);
  }
  // staging b is free once its previous copy-out (two calls ago) has finished
  CK(cudaStreamWaitEvent(st, ev_dpushed_[b], 0));
  // DMA of the expected size: the largest of the last applied deltas + 25%
  // (the whole capacity until one was seen); the pack writes bytes past it
  // into the host buffer itself (no kernel on the copy-out stream: it would
  // share a hardware queue with other streams' work)
  size_t est = cap;
  if (delta_seen_ > 0) {
    size_t m = 0;
    for (const auto& v : delta_recent_) m = std::max(m, v.load(std::memory_order_relaxed));
    est = std::min(cap, (m + m / 4 + 65536 + 15) / 16 * 16);
  }
  DeltaArgs a{};
  a.out = r.out.as<float>();
  a.idx = r.idx;
  a.count = counts_.as<int32_t>() + r.count_slot;
  a.cnt_stride = cnt_stride_;
  a.dst = delta_stage_[b].as<uint8_t>();
  a.host = static_cast<uint8_t*>(dptr);
  a.copied = static_cast<long long>(est);
  a.Cs = r.Cs, a.S = S_;
  a.HW = static_cast<long long>(r.d.H) * r.d.W;
  launch_pack_delta(a, st);
  CK(cudaEventRecord(ev_dstaged_[b], st));
  CK(cudaStreamWaitEvent(ctx_->d2h, ev_dstaged_[b], 0));
  CK(cudaMemcpyAsync(host_buf, delta_stage_[b].p, est, cudaMemcpyDeviceToHost, ctx_->d2h));
  delta_dma_last_ = est;
  CK(cudaEventRecord(ev_dpushed_[b], ctx_->d2h));
  cudaEvent_t ev;
  {
    std::lock_guard<std::mutex> lk(delta_mu_);
    DeltaCopy& dc = delta_host_[host_buf];
    if (!dc.ev) CK(cudaEventCreateWithFlags(&dc.ev, cudaEventDisableTiming));
    ev = dc.ev;
  }
  CK(cudaEventRecord(ev, ctx_->d2h));
}

void Net::apply_output_delta(int node, const void* host_buf, float* mirror, int s0, int s1) {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size())) throw_invalid("apply_output_delta: bad node");
  if (s0 < 0 || s1 > S_ || s0 > s1) throw_invalid("apply_output_delta: bad stream range");
  cudaEvent_t ev;
  {
    std::lock_guard<std::mutex> lk(delta_mu_);
    auto it = delta_host_.find(host_buf);
    if (it == delta_host_.end()) throw_invalid("apply_output_delta: no delta was copied into this buffer");
    ev = it->second.ev;
  }
  CK(cudaEventSynchronize(ev));
  const NodeRT& r = nodes_[node];
  const int Cs = r.Cs;
  const uint8_t* buf = static_cast<const uint8_t*>(host_buf);
  const int32_t* hdr = reinterpret_cast<const int32_t*>(buf);
  size_t off = delta_header_bytes(S_);
  const size_t HWC = static_cast<size_t>(r.d.H) * r.d.W * Cs;
  for (int s = 0; s < s1; ++s) {
    const int n = hdr[s];
    if (s >= s0) {
      const int32_t* ids = reinterpret_cast<const int32_t*>(buf + off);
      const float* vals = reinterpret_cast<const float*>(buf + off + (static_cast<size_t>(n) * 4 + 15) / 16 * 16);
      float* m = mirror + s * HWC;
      for (int k = 0; k < n; ++k)
        std::memcpy(m + static_cast<size_t>(ids[k]) * Cs, vals + static_cast<size_t>(k) * Cs, Cs * 4);
    }
    off += delta_stream_bytes(n, Cs);
  }
  if (s1 == S_) {  // the whole buffer's size feeds the next DMA estimates
    for (int s = s1; s < S_; ++s) off += delta_stream_bytes(hdr[s], Cs);
    delta_recent_[delta_seen_.fetch_add(1) % 4].store(off, std::memory_order_relaxed);
  }
}

void Net::set_external(const float* x_chw, const uint8_t* map, const int32_t* rowcol, int64_t n, bool full) {
  NodeRT& e = nodes_[0];
  const NodeDesc& d = e.d;
  cudaStream_t st = ctx_->stream;
  const size_t HW = static_cast<size_t>(d.H) * d.W;
  // running bound of the uploaded values (the consumer's state holds earlier uploads too)
  {
    float m = ext_amax_[0];
    const size_t n_el = static_cast<size_t>(d.C) * HW;
    for (size_t k = 0; k < n_el; ++k) m = std::max(m, std::fabs(x_chw[k]));
    ext_amax_[0] = m;
    CK(cudaMemcpyAsync(amax_entry(0), &ext_amax_[0], sizeof(float), cudaMemcpyHostToDevice, st));
  }
  // the frame of the external node is a CHW staging copy
  CK(cudaMemcpyAsync(frame_.p, x_chw, static_cast<size_t>(d.C) * HW * sizeof(float), cudaMemcpyHostToDevice, st));
  launch_chw_to_nhwc(frame_.as<float>(), e.out.as<float>(), d.C, e.Cs, static_cast<int>(HW), st);
  // the upstream map as a bitmap (common.cuh); full: a forced full update sees
  // every upstream pixel as changed (a Reuse1x1 layer then recomputes
  // everything, layers.cpp:64-71)
  const int nw = (d.W + 31) / 32;
  std::vector<uint32_t> m(static_cast<size_t>(d.H) * nw, 0u);
  for (int row = 0; row < d.H; ++row)
    for (int col = 0; col < d.W; ++col)
      if (full || (map && map[static_cast<size_t>(row) * d.W + col])) m[static_cast<size_t>(row) * nw + (col >> 5)] |= 1u << (col & 31);
  // ordered on the ctx stream after the previous frame's kernels, which may
  // still read the map, list and count (pageable sources are staged at call time)
  CK(cudaMemcpyAsync(e.outmap, m.data(), m.size() * 4, cudaMemcpyHostToDevice, st));
  std::vector<int32_t> idx;
  if (full) {
    idx.resize(HW);
    for (size_t k = 0; k < HW; ++k) idx[k] = static_cast<int32_t>(k);
    CK(cudaMemcpyAsync(e.idx, idx.data(), HW * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  } else if (rowcol) {
    idx.resize(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) idx[k] = rowcol[2 * k] * d.W + rowcol[2 * k + 1];
    if (n) CK(cudaMemcpyAsync(e.idx, idx.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  const int32_t cnt = static_cast<int32_t>(full ? HW : rowcol ? n : 0);
  CK(cudaMemcpyAsync(counts_.as<int32_t>() + e.count_slot, &cnt, sizeof(cnt), cudaMemcpyHostToDevice, st));
}

void Net::reset(int stream) {
  if (stream < -1 || stream >= S_) throw_invalid("reset: stream out of range");
  cudaStream_t st = ctx_->stream;
  const int s0 = stream < 0 ? 0 : stream, s1 = stream < 0 ? S_ : stream + 1;
  for (int k = s0; k < s1; ++k) s8_pending_[k] = 1;
  for (NodeRT& r : nodes_) {
    if (r.d.kind == kExternal) continue;
    const size_t per_out = r.out.bytes / S_;
    CK(cudaMemsetAsync(static_cast<uint8_t*>(r.out.p) + per_out * s0, 0, per_out * (s1 - s0), st));
    if (r.state.bytes) {
      const size_t per = r.state.bytes / S_;
      CK(cudaMemsetAsync(static_cast<uint8_t*>(r.state.p) + per * s0, 0, per * (s1 - s0), st));
    }
  }
  CK(cudaMemsetAsync(boot_req_.as<uint8_t>() + s0, 1, s1 - s0, st));
  for (int e = 0; e <= static_cast<int>(nodes_.size()); ++e)
    CK(cudaMemsetAsync(amax_.as<float>() + static_cast<size_t>(e) * S_ + s0, 0, (s1 - s0) * sizeof(float), st));
  for (int k = s0; k < s1; ++k) ext_amax_[k] = 0.0f;
}

// Upload the per-stream thresholds and OR `rescan` into the device requests.
void Net::upload_taus(const std::vector<uint8_t>& rescan) {
  cudaStream_t st = ctx_->stream;
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(taus_.p, stream_taus_.data(), stream_taus_.size() * sizeof(float), cudaMemcpyHostToDevice));
  std::vector<uint8_t> cur(nodes_.size());
  CK(cudaMemcpy(cur.data(), rescan_req_.p, nodes_.size(), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < cur.size(); ++i) cur[i] |= rescan[i];
  CK(cudaMemcpy(rescan_req_.p, cur.data(), nodes_.size(), cudaMemcpyHostToDevice));
}

void Net::set_thresholds(const std::vector<float>& taus) {
  std::vector<int> conv_nodes;
  for (size_t i = 0; i < nodes_.size(); ++i)
    if (nodes_[i].d.kind == CBG_LAYER_CONV) conv_nodes.push_back(static_cast<int>(i));
  if (taus.size() != conv_nodes.size()) throw_invalid("set_thresholds: expected one tau per conv layer");
  for (float t : taus)
    if (!(t >= 0.0f)) throw_invalid("set_thresholds: tau must be >= 0");
  std::vector<uint8_t> rescan(nodes_.size(), 0);
  for (size_t k = 0; k < conv_nodes.size(); ++k) {
    const int i = conv_nodes[k];
    // Sparse detection is exact only while tau does not decrease:
    // a lowered threshold re-detects every pixel once.
    for (int s = 0; s < S_; ++s) {
      float& cur = stream_taus_[static_cast<size_t>(i) * S_ + s];
      if (taus[k] < cur) rescan[i] = 1;
      cur = taus[k];
    }
    host_taus_[i] = taus[k];
    nodes_[i].d.tau = taus[k];
  }
  upload_taus(rescan);
}

void Net::set_stream_thresholds(int stream, const std::vector<float>& taus) {
  if (stream < 0 || stream >= S_) throw_invalid("set_stream_thresholds: stream out of range");
  std::vector<int> conv_nodes;
  for (size_t i = 0; i < nodes_.size(); ++i)
    if (nodes_[i].d.kind == CBG_LAYER_CONV) conv_nodes.push_back(static_cast<int>(i));
  if (taus.size() != conv_nodes.size()) throw_invalid("set_stream_thresholds: expected one tau per conv layer");
  for (float t : taus)
    if (!(t >= 0.0f)) throw_invalid("set_stream_thresholds: tau must be >= 0");
  std::vector<uint8_t> rescan(nodes_.size(), 0);
  for (size_t k = 0; k < conv_nodes.size(); ++k) {
    float& cur = stream_taus_[static_cast<size_t>(conv_nodes[k]) * S_ + stream];
    if (taus[k] < cur) rescan[conv_nodes[k]] = 1;  // (dense re-detection of the node, all streams: exact)
    cur = taus[k];
  }
  upload_taus(rescan);
}

std::vector<float> Net::thresholds() const {
  std::vector<float> t;
  for (const NodeRT& r : nodes_)
    if (r.d.kind == CBG_LAYER_CONV) t.push_back(host_taus_[&r - nodes_.data()]);
  return t;
}

void Net::set_dense(bool dense) {
  dense_ = dense;
  const uint8_t v = dense ? 1 : 0;
  CK(cudaMemcpyAsync(dense_flag_.p, &v, 1, cudaMemcpyHostToDevice, ctx_->stream));
  CK(cudaStreamSynchronize(ctx_->stream));
}

void Net::read_output(int node, int stream, float* out_chw) {
  if (node < 0) node = static_cast<int>(nodes_.size()) - 1;
  if (node >= static_cast<int>(nodes_.size()) || stream < 0 || stream >= S_) throw_invalid("read_output: bad node/stream");
  const NodeRT& r = nodes_[node];
  const size_t HW = static_cast<size_t>(r.d.H) * r.d.W;
  DevBuf tmp;
  tmp.alloc(static_cast<size_t>(r.d.C) * HW * sizeof(float));
  launch_nhwc_to_chw(r.out.as<float>() + static_cast<size_t>(stream) * HW * r.Cs, tmp.as<float>(), r.d.C, r.Cs,
                     static_cast<int>(HW), ctx_->stream);
  CK(cudaMemcpyAsync(out_chw, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, ctx_->stream));
  CK(cudaStreamSynchronize(ctx_->stream));
}

void Net::read_state(int node, int stream, float* out_chw) {
  if (node < 0 || node >= static_cast<int>(nodes_.size()) || stream < 0 || stream >= S_)
    throw_invalid("read_state: bad node/stream");
  const NodeRT& r = nodes_[node];
  if (!r.state.bytes) throw_invalid("read_state: node has no input state (not a detect-policy conv)");
  const size_t HW = static_cast<size_t>(r.d.Hi) * r.d.Wi;
  if (r.state_chw) {
    CK(cudaMemcpyAsync(out_chw, r.state.as<float>() + static_cast<size_t>(stream) * HW * r.d.Ci,
                       static_cast<size_t>(r.d.Ci) * HW * sizeof(float), cudaMemcpyDeviceToHost, ctx_->stream));
    CK(cudaStreamSynchronize(ctx_->stream));
    return;
  }
  DevBuf tmp;
  tmp.alloc(static_cast<size_t>(r.d.Ci) * HW * sizeof(float));
  launch_nhwc_to_chw(r.state.as<float>() + static_cast<size_t>(stream) * HW * r.Csi, tmp.as<float>(), r.d.Ci, r.Csi,
                     static_cast<int>(HW), ctx_->stream);
  CK(cudaMemcpyAsync(out_chw, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, ctx_->stream));
  CK(cudaStreamSynchronize(ctx_->stream));
}

void Net::read_counts(std::vector<int32_t>& counts) {
  counts.resize(static_cast<size_t>(cnt_stride_) * S_);
  CK(cudaMemcpyAsync(counts.data(), counts_.p, counts.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx_->stream));
  CK(cudaStreamSynchronize(ctx_->stream));
}

int64_t Net::count_of(const std::vector<int32_t>& counts, int node, int stream, bool worst) const {
  const NodeRT& r = nodes_[node];
  const int slot = worst ? r.wc_slot : r.count_slot;
  if (slot < 0) return -1;
  return counts[static_cast<size_t>(stream) * cnt_stride_ + slot];
}

void Net::read_changes(int node, int stream, uint8_t* map, int32_t* rowcol, int64_t* count, bool worst) {
  if (node < 0 || node >= static_cast<int>(nodes_.size()) || stream < 0 || stream >= S_)
    throw_invalid("read_changes: bad node/stream");
  const NodeRT& r = nodes_[node];
  std::vector<int32_t> counts;
  read_counts(counts);
  const size_t HW = static_cast<size_t>(r.d.H) * r.d.W;
  int64_t n = count_of(counts, node, stream, worst);
  if (worst && r.d.inputs[0] < 0) n = count_of(counts, node, stream, false);  // first layer: own map
  const int32_t* didx = (worst && r.d.inputs[0] >= 0) ? r.wc_idx.as<int32_t>() : r.idx;
  std::vector<int32_t> idx(static_cast<size_t>(std::max<int64_t>(n, 0)));
  if (n > 0)
    CK(cudaMemcpy(idx.data(), didx + static_cast<size_t>(stream) * HW, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  // the device list is row-major per compaction tile, tiles in completion
  // order; the reference's list (change.cpp:77-84) is row-major overall
  std::sort(idx.begin(), idx.end());
  if (count) *count = n;
  if (map) {
    std::memset(map, 0, HW);
    for (int32_t p : idx) map[p] = 1;
  }
  if (rowcol)
    for (int64_t k = 0; k < n; ++k) {
      rowcol[2 * k] = idx[k] / r.d.W;
      rowcol[2 * k + 1] = idx[k] % r.d.W;
    }
}

}  // namespace cbg
