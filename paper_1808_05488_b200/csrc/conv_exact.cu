// conv_exact.cu — change-based convolution update for narrow layers on the CUDA
// cores, bit-identical to the reference.
//
// Replaces, for layers with few output channels (Cout <= 16: the first and last
// layer of the scene-labeling net), the partial im2col + gemm + update_output
// of the reference (dense.cpp:44-112, layers.cpp:10-31):
//
//   for every changed output pixel p (index list and count on device)
//     acc[o] = 0;  for r ascending: acc[o] = acc[o] + K[o][r] * X[r][p]
//     prev_output[p][o] = act(acc[o] + b[o])
//
// with r = (c*kh + kj)*kw + ki (im2col row order, dense.cpp:69-79), one IEEE
// rounding after every multiply and every add (the reference is built without
// FMA contraction: __fmul_rn / __fadd_rn are never fused by nvcc), zeros for
// taps outside the input (they are added too, as the reference does), and
// act = (v < 0) ? 0 : v (std::max(v, 0.f)). The results are therefore
// bit-identical to the reference's sequential fp32 GEMM, not merely close.
//
// Why CUDA cores: a tcgen05 MMA has N >= 16 and pays a per-K-block gather and
// tf32 split that dominate when Cout is 8 or 16. Here one
// thread owns one changed pixel and G output channels: per K-row it does one
// (L1-cached) input load, G/4 shared-memory float4 weight broadcasts and G
// multiply/add pairs, so the FP32 pipe does the work.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace cbg {

namespace {

constexpr int kThreads = 128;

constexpr int kPix = 2;
constexpr int kMaxStreams = 1024;  // changed pixels per thread (each weight broadcast feeds both)

// Packed fp32x2 arithmetic (sm_100 FMUL2 / FFMA2): two lanes per instruction.
// mul.rn rounds each product like the reference's `kr[o] * xv`; the add is an
// fma with a multiplier of 1.0 that ptxas cannot see (`one` is a kernel
// argument), i.e. RN(acc * 1 + prod) = RN(acc + prod), the reference's
// `acc[o] += ...`. A plain add.rn.f32x2 after mul.rn.f32x2 is contracted into
// FFMA2 by ptxas (one rounding: not the reference's result).
CBG_DEV unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
CBG_DEV void f2_unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
CBG_DEV unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
CBG_DEV unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// One kernel row (KW taps of one input channel and kernel row) of the sum for
// kPix pixels; acc holds output-channel pairs.
template <int G, int KW>
CBG_DEV void exact_row(unsigned long long (&acc)[kPix][G / 2], const float (&xv)[kPix][KW], const float4* w4,
                       unsigned long long one) {
#pragma unroll
  for (int ki = 0; ki < KW; ++ki) {
    unsigned long long xx[kPix];
#pragma unroll
    for (int u = 0; u < kPix; ++u) xx[u] = f2_pack(xv[u][ki], xv[u][ki]);
#pragma unroll
    for (int q = 0; q < G / 4; ++q) {
      const float4 w = w4[ki * (G / 4) + q];
      const unsigned long long w01 = f2_pack(w.x, w.y), w23 = f2_pack(w.z, w.w);
#pragma unroll
      for (int u = 0; u < kPix; ++u) {
        acc[u][2 * q + 0] = f2_fma(acc[u][2 * q + 0], one, f2_mul(w01, xx[u]));
        acc[u][2 * q + 1] = f2_fma(acc[u][2 * q + 1], one, f2_mul(w23, xx[u]));
      }
    }
  }
}

// G output channels per thread, KW = kernel width (compile time, so a kernel
// row's KW inputs are loaded together and the next row is prefetched while the
// current one is summed). CHECK = false when every tap of every valid output
// pixel lies inside the input (padding 0), which drops the bounds tests.
// PS = pixel stride of the source when known at compile time (1: CHW planes),
// 0 = runtime a.pstride (NHWC).
//
// Work is the concatenation of all streams' index lists (per-stream prefix of
// the device counts, computed per CTA), split into blocks of kThreads*kPix
// pixels that the persistent grid strides over, so uneven streams balance.
template <int G, int KW, bool CHECK, int PS>
// <= 88 registers: a 128-thread CTA (11k) still fits beside a resident GEMM CTA
__global__ void __maxnreg__(88) conv_exact_kernel(ConvExactArgs a) {  // launched with kThreads = 128
  CBG_PDL_ENTRY;
  extern __shared__ __align__(16) float sw[];  // [K][G] weights of this output group, reference r order
  __shared__ int s_prefix[kMaxStreams + 1];
  const int og = blockIdx.y;  // output-channel group
  const int K = a.Cin * a.kh * KW;
  // weights [Cout][K] row-major -> [K][G]: all of a thread's loads first (one
  // memory latency per CTA, not one per element)
  {
    constexpr int kU = 8;
    for (int i0 = 0; i0 < K * G; i0 += kU * kThreads) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads + threadIdx.x;
        const int r = i / G, o = og * G + (i - r * G);
        v[u] = (i < K * G && o < a.Cout) ? __ldg(a.w + static_cast<long long>(o) * K + r) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kThreads + threadIdx.x;
        if (i < K * G) sw[i] = v[u];
      }
    }
  }
  if (threadIdx.x < 32) {  // block counts: ceil(count / (kThreads*kPix)) per stream, exclusive prefix
    const int lane = threadIdx.x;
    int carry = 0;
    if (lane == 0) s_prefix[0] = 0;
    for (int s0 = 0; s0 < a.S; s0 += 32) {
      const int s = s0 + lane;
      const int v = s < a.S ? (a.count[s * a.cnt_stride] + kThreads * kPix - 1) / (kThreads * kPix) : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (s < a.S) s_prefix[s + 1] = carry + inc;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  const int total = s_prefix[a.S];
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  const float4* sw4 = reinterpret_cast<const float4*>(sw);
  const int ps = PS ? PS : a.pstride;
  const long long rstride = static_cast<long long>(a.Win) * ps;
  for (int wb = blockIdx.x; wb < total; wb += gridDim.x) {
    float vmax = 0.0f;
    int lo = 0, hi = a.S;  // stream s with s_prefix[s] <= wb < s_prefix[s+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_prefix[mid] <= wb) lo = mid;
      else hi = mid;
    }
    const int s = lo;
    const int n = a.count[s * a.cnt_stride];
    const int kb = (wb - s_prefix[s]) * (kThreads * kPix) + threadIdx.x;
    const float* src = a.src + static_cast<long long>(s) * a.src_sstride;
    const int32_t* list = a.idx + static_cast<long long>(s) * HWo;
    float* out = a.out + static_cast<long long>(s) * HWo * a.Co4;
    // pixel u of this thread: list entry kb + u*kThreads (lanes stay coalesced)
    int p[kPix], j0[kPix];
    const float* base[kPix];
    uint32_t colok[kPix];
#pragma unroll
    for (int u = 0; u < kPix; ++u) {
      const int k = kb + u * kThreads;
      p[u] = k < n ? list[k] : -1;
      const int pp = p[u] < 0 ? 0 : p[u];
      const int jo = pp / a.Wout, io = pp - jo * a.Wout;
      j0[u] = jo * a.stride - a.pad;
      const int i0 = io * a.stride - a.pad;
      base[u] = src + static_cast<long long>(j0[u]) * rstride + static_cast<long long>(i0) * ps;
      colok[u] = 0;
      if (CHECK) {
#pragma unroll
        for (int ki = 0; ki < KW; ++ki)
          colok[u] |= static_cast<uint32_t>(static_cast<unsigned>(i0 + ki) < static_cast<unsigned>(a.Win)) << ki;
      }
    }
    // kernel rows in r order: (c, kj) -> offset c*cstride + kj*rstride, advanced incrementally
    auto load_row = [&](long long off, int kj, float (&xv)[kPix][KW]) {
#pragma unroll
      for (int u = 0; u < kPix; ++u) {
        const float* sp = base[u] + off;
        if (CHECK) {
          const bool row_ok = static_cast<unsigned>(j0[u] + kj) < static_cast<unsigned>(a.Hin);
#pragma unroll
          for (int ki = 0; ki < KW; ++ki)
            xv[u][ki] = (row_ok && ((colok[u] >> ki) & 1u)) ? __ldg(sp + ki * ps) : 0.0f;
        } else {
#pragma unroll
          for (int ki = 0; ki < KW; ++ki) xv[u][ki] = __ldg(sp + ki * ps);
        }
      }
    };
    const long long cwrap = a.cstride - static_cast<long long>(a.kh) * rstride;
    long long off = 0;
    int kj = 0;
    auto advance = [&]() {
      off += rstride;
      if (++kj == a.kh) {
        kj = 0;
        off += cwrap;
      }
    };
    unsigned long long acc[kPix][G / 2];
#pragma unroll
    for (int u = 0; u < kPix; ++u)
#pragma unroll
      for (int o = 0; o < G / 2; ++o) acc[u][o] = 0ull;  // +0.0f pairs
    const unsigned long long one = a.one_x2;
    if constexpr (KW == 1 && PS == 0 && !CHECK) {
      if (a.kh == 1 && a.cstride == 1) {
        // 1x1 on NHWC: r = c, a pixel's channel vector is contiguous and
        // 16-B aligned (Cs % 4 == 0): float4 loads, 4 K-rows each, 2 ahead
        const int nc4 = (a.Cin + 3) >> 2;
        float4 xq[3][kPix];
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
          for (int u = 0; u < kPix; ++u)
            xq[d][u] = d < nc4 ? ldg_nc_f4(base[u] + 4 * d) : make_float4(0.f, 0.f, 0.f, 0.f);
        int c4 = 0;
        for (; c4 < nc4; ++c4) {
#pragma unroll
          for (int u = 0; u < kPix; ++u)
            xq[2][u] = c4 + 2 < nc4 ? ldg_nc_f4(base[u] + 4 * (c4 + 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
          const int rem = a.Cin - 4 * c4;  // real channels in this group (tail: < 4)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e < rem) {
              float xv[kPix][1];
#pragma unroll
              for (int u = 0; u < kPix; ++u) xv[u][0] = (&xq[0][u].x)[e];
              exact_row<G, 1>(acc, xv, sw4 + (4 * c4 + e) * (G / 4), one);
            }
          }
#pragma unroll
          for (int u = 0; u < kPix; ++u) {
            xq[0][u] = xq[1][u];
            xq[1][u] = xq[2][u];
          }
        }
        goto epilogue;
      }
    }
    {
    const int rows = a.Cin * a.kh;  // (c, kj) kernel rows, in the reference's r order
    float xa[kPix][KW], xb[kPix][KW];
    load_row(off, kj, xa);
    advance();
    int row = 0;
    for (; row + 2 <= rows; row += 2) {
      load_row(off, kj, xb);
      advance();
      exact_row<G, KW>(acc, xa, sw4 + row * KW * (G / 4), one);
      if (row + 2 < rows) {
        load_row(off, kj, xa);
        advance();
      }
      exact_row<G, KW>(acc, xb, sw4 + (row + 1) * KW * (G / 4), one);
    }
    if (row < rows) exact_row<G, KW>(acc, xa, sw4 + row * KW * (G / 4), one);
    }
  epilogue:
#pragma unroll
    for (int u = 0; u < kPix; ++u) {
      if (p[u] < 0) continue;
      float* orow = out + static_cast<long long>(p[u]) * a.Co4 + og * G;
#pragma unroll
      for (int q = 0; q < G / 4; ++q) {
        const int o = og * G + 4 * q;
        if (o < a.Co4) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float alo, ahi;
            f2_unpack(acc[u][2 * q + (e >> 1)], alo, ahi);
            float y = __fadd_rn((e & 1) ? ahi : alo, o + e < a.Cout ? __ldg(a.bias + o + e) : 0.0f);
            if (a.relu) y = (y < 0.0f) ? (a.slope != 0.0f ? y * a.slope : 0.0f) : y;  // std::max(v, 0.f) / leaky
            v[e] = o + e < a.Cout ? y : 0.0f;
            vmax = fmaxf(vmax, fabsf(v[e]));
          }
          *reinterpret_cast<float4*>(orow + 4 * q) = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    }
    warp_amax(a.amax_out ? a.amax_out + s : nullptr, vmax);
  }
}

template <int G, int KW, bool CHECK, int PS>
void launch_k(const ConvExactArgs& a, cudaStream_t st) {
  const int K = a.Cin * a.kh * a.kw;
  const size_t smem = static_cast<size_t>(K) * G * sizeof(float);
  static int per_sm = 0;
  static size_t per_sm_smem = 0;
  if (per_sm == 0 || per_sm_smem != smem) {
    cudaFuncSetAttribute(conv_exact_kernel<G, KW, CHECK, PS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         232448 - 8192);  // leaves room for the static s_prefix
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_exact_kernel<G, KW, CHECK, PS>, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    per_sm_smem = smem;
  }
  // persistent: every CTA resident, striding over the blocks of all streams
  static const int cap = std::getenv("CBG_EXACT_PER_SM") ? std::atoi(std::getenv("CBG_EXACT_PER_SM")) : 0;
  const int psm = cap > 0 ? std::min(cap, per_sm) : per_sm;
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  long long bx = static_cast<long long>(a.sm_count) * psm;
  const long long most = ((HWo + kThreads * kPix - 1) / (kThreads * kPix)) * a.S;
  if (bx > most) bx = most;
  if (bx < 1) bx = 1;
  dim3 grid(static_cast<unsigned>(bx), (a.Cout + G - 1) / G);
  launch_k(conv_exact_kernel<G, KW, CHECK, PS>, grid, dim3(kThreads), smem, st, a);
}

template <int G, int KW>
void launch_gk(const ConvExactArgs& a, cudaStream_t st) {
  // every tap of every valid output pixel inside the input (padding 0 and
  // output dims not pinned beyond the derived ones): no bounds tests
  const bool inside = a.pad == 0 && (a.Hout - 1) * a.stride + a.kh <= a.Hin &&
                      (a.Wout - 1) * a.stride + a.kw <= a.Win;
  if (a.pstride == 1) {
    if (inside) launch_k<G, KW, false, 1>(a, st);
    else launch_k<G, KW, true, 1>(a, st);
  } else {
    if (inside) launch_k<G, KW, false, 0>(a, st);
    else launch_k<G, KW, true, 0>(a, st);
  }
}

template <int G>
void launch_g(const ConvExactArgs& a, cudaStream_t st) {
  switch (a.kw) {
    case 1: launch_gk<G, 1>(a, st); break;
    case 2: launch_gk<G, 2>(a, st); break;
    case 3: launch_gk<G, 3>(a, st); break;
    case 4: launch_gk<G, 4>(a, st); break;
    case 5: launch_gk<G, 5>(a, st); break;
    case 6: launch_gk<G, 6>(a, st); break;
    case 7: launch_gk<G, 7>(a, st); break;
    case 8: launch_gk<G, 8>(a, st); break;
    case 9: launch_gk<G, 9>(a, st); break;
    case 11: launch_gk<G, 11>(a, st); break;
    default: break;  // exact_supported() keeps other widths on the tcgen05 path
  }
}

}  // namespace

bool conv_exact_supported(int kw) { return (kw >= 1 && kw <= 9) || kw == 11; }

int conv_exact_group(int cout) { return cout <= 4 ? 4 : cout <= 8 ? 8 : 16; }

size_t conv_exact_smem_bytes(int cout, int K) {
  return static_cast<size_t>(K) * conv_exact_group(cout) * sizeof(float);
}

void launch_conv_exact(const ConvExactArgs& a, cudaStream_t st) {
  switch (conv_exact_group(a.Cout)) {
    case 4: launch_g<4>(a, st); break;
    case 8: launch_g<8>(a, st); break;
    default: launch_g<16>(a, st); break;
  }
}

}  // namespace cbg
