// change_kernels.cu — HBM-bound kernels of the CBinfer hot path (sm_100a).
//
//   detect_frame    fused frame ingest (CHW) + thresholded change detection +
//                   closed-loop state update        ref change.cpp:20-43
//   detect_list     the same on NHWC inputs, walking only the producer's
//                   update set                      ref change.cpp:20-43
//   dilate_compact  window dilation of (OR-ed) change bitmaps fused with the
//                   stream compaction into the index list (one warp per
//                   band of rows, row-major runs placed by one atomicAdd
//                   each), optionally with a following 2x2 pool's map/list
//                                                   ref change.cpp:45-84
//   pool            change-based max pooling       ref layers.cpp:148-179
//   join            Add / Concat at changed pixels  ref network.cpp:364-398
//
// Arithmetic is exact IEEE fp32 (no fast-math): |x - s| > tau and the max
// comparisons are bit-identical to the reference.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace cbg {

namespace {

constexpr int kThreads = 256;
// The 4-pixel frame-ingest kernels hold 8 float4 per thread (~80 registers):
// 128-thread CTAs (10k registers) still fit on an SM beside a resident GEMM
// CTA of another stream group (672 x 80 of the 64k registers).
constexpr int kFrameThreads = 128;

int blocks_for(long long work, int per_block, int S, int sm_count) {
  long long b = (work + per_block - 1) / per_block;
  long long cap = (static_cast<long long>(sm_count) * 8 + S - 1) / S;  // ~8 CTAs/SM in total
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// CTAs per stream (grid.x) of a grid-stride kernel: enough for the work, and at
// most one whole wave of the kernel's resident CTAs over all streams (CBG_WAVES
// = n: n waves), so no launch ends with a sliver of a wave on a few SMs
// (blocks_for's fixed 8 CTAs per SM left 2.05 waves of the 8-bit detect at 64
// streams: SMs idle 22% of the launch) and each thread's iterations even out.
// CBG_WAVE_GRID=0: blocks_for.
template <class... Args>
int wave_grid(void (*kernel)(Args...), int threads, long long work, int per_cta, int S, int legacy_mult) {
  static const bool on = !(std::getenv("CBG_WAVE_GRID") && std::atoi(std::getenv("CBG_WAVE_GRID")) == 0);
  static const int waves = std::getenv("CBG_WAVES") ? std::max(1, std::atoi(std::getenv("CBG_WAVES"))) : 1;
  if (!on) return legacy_mult * blocks_for(work, per_cta * legacy_mult, S, sm_count());
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ_cache;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), threads);
    auto it = occ_cache.find(key);
    if (it == occ_cache.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        occ = 1;
      }
      it = occ_cache.emplace(key, occ).first;
    }
    occ = it->second;
  }
  const long long need = (work + per_cta - 1) / per_cta;
  const long long cap = std::max(1LL, static_cast<long long>(waves) * occ * sm_count() / S);
  return static_cast<int>(std::max(1LL, std::min(need, cap)));
}

// ---------------------------------------------------------------------------
// Change-map output of the detect kernels (bitmaps, common.cuh).
// ---------------------------------------------------------------------------
// One 4-pixel group q (pixels 4q..4q+3), bit j of ch = pixel 4q+j changed,
// into a map begin_frame cleared. plain (W % 32 == 0): the 8 groups of a word
// are 8 consecutive lanes (group ids are lane-aligned), so a warp with any
// change OR-s each word over its 8 lanes with shuffles and stores it whole
// (the word belongs to those lanes alone); the common all-unchanged warp pays
// one vote. Otherwise (a group may straddle rows) changed pixels are OR-ed in
// one by one. Every lane of the warp must call it (warp-uniform loop trips).
CBG_DEV void put_quad(uint32_t* m, long long q, bool valid, uint32_t ch, int W, int plain) {
  if (!__any_sync(0xffffffffu, ch != 0u)) return;
  if (plain) {
    uint32_t v = ch << (4 * (threadIdx.x & 7));
    v |= __shfl_xor_sync(0xffffffffu, v, 1);
    v |= __shfl_xor_sync(0xffffffffu, v, 2);
    v |= __shfl_xor_sync(0xffffffffu, v, 4);
    if (valid && v && (threadIdx.x & 7) == 0) m[q >> 3] = v;
  } else if (valid && ch) {
    for (int j = 0; j < 4; ++j)
      if ((ch >> j) & 1u) map_set(m, (q << 2) + j, W);
  }
}

// detected-pixel count of a stream (dc: its counter): one atomicAdd per CTA
// (warp sums combined in shared memory), plus every pixel on a full update.
// Every thread of the CTA must call it.
CBG_DEV void detect_count(int32_t* dc, int nch, bool boot, long long HW) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  nch = __reduce_add_sync(0xffffffffu, nch);
  if ((threadIdx.x & 31) == 0 && nch) atomicAdd(&s_cnt, nch);
  __syncthreads();
  if (threadIdx.x == 0 && dc) {
    const int v = s_cnt + ((boot && blockIdx.x == 0) ? static_cast<int>(HW) : 0);
    if (v) atomicAdd(dc, v);
  }
}

// ---------------------------------------------------------------------------
// detect on the network-input frame. One thread per pixel: the C channel
// planes are read coalesced, the NHWC state as one 16-B vector per 4 channels.
// ---------------------------------------------------------------------------
template <bool kVec4>
__global__ void __launch_bounds__(kThreads) detect_frame_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const float* x = *a.x_slot + static_cast<long long>(s) * a.x_sstride;
  float* st = a.state + static_cast<long long>(s) * HW * a.Cs;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  const int lane = threadIdx.x & 31;
  float vmax = 0.0f;
  int nch = 0;
  if constexpr (kVec4) {
    // C <= 4 (Cs == 4), HW % 4 == 0: one thread = 4 consecutive pixels; the C
    // planes are read as float4, the 4 NHWC state vectors as 4 float4.
    const long long n4 = HW >> 2;
    for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q - lane < n4;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
      const bool valid = q < n4;
      uint32_t ch = 0;
      if (valid) {
        const long long p0 = q << 2;
        float4 xv[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          xv[c] = c < a.C ? ldg_nc_f4(x + c * HW + p0) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 sv[4];
        if (!boot) {
#pragma unroll
          for (int j = 0; j < 4; ++j) sv[j] = *reinterpret_cast<const float4*>(st + (p0 + j) * 4);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float px[4] = {(&xv[0].x)[j], (&xv[1].x)[j], (&xv[2].x)[j], (&xv[3].x)[j]};
          bool changed = false;
          if (!boot) {
            const float sp[4] = {sv[j].x, sv[j].y, sv[j].z, sv[j].w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c < a.C) changed |= fabsf(px[c] - sp[c]) > tau;
          }
          if (changed || write_all) {
            *reinterpret_cast<float4*>(st + (p0 + j) * 4) = make_float4(px[0], px[1], px[2], px[3]);
            vmax = fmaxf(vmax, fmaxf(fmaxf(fabsf(px[0]), fabsf(px[1])), fmaxf(fabsf(px[2]), fabsf(px[3]))));
          }
          ch |= static_cast<uint32_t>(changed) << j;
        }
      }
      put_quad(m, q, valid, ch, a.W, a.map_plain);
      nch += __popc(ch);
    }
  } else {
    for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < HW;
         p += static_cast<long long>(gridDim.x) * blockDim.x) {
      float* sp = st + p * a.Cs;
      bool changed = false;
      if (!boot) {
        for (int c0 = 0; c0 < a.Cs; c0 += 4) {
          const float4 sv = *reinterpret_cast<const float4*>(sp + c0);
          const float s4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = c0 + j;
            if (c < a.C) changed |= fabsf(__ldg(x + c * HW + p) - s4[j]) > tau;
          }
        }
        if (changed) {
          map_set(m, p, a.W);
          ++nch;
        }
      }
      if (changed || write_all) {
        for (int c0 = 0; c0 < a.Cs; c0 += 4) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            v[j] = (c0 + j < a.C) ? __ldg(x + (c0 + j) * HW + p) : 0.0f;
            vmax = fmaxf(vmax, fabsf(v[j]));
          }
          *reinterpret_cast<float4*>(sp + c0) = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    }
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// ---------------------------------------------------------------------------
// detect on the network-input frame against a CHW (planar, unpadded) state:
// the layout of the first layer's state when that layer runs the CUDA-core
// path (conv_exact.cu reads its taps from the planes). Every byte moved is
// algorithmic: 4*C B of frame + 4*C B of state per pixel, state written only
// where a pixel of the 4-pixel group changed. One thread = 4 consecutive
// pixels (HW % 4 == 0), C <= 4 kept in registers.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFrameThreads) detect_frame_chw_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const float* x = *a.x_slot + static_cast<long long>(s) * a.x_sstride;
  float* st = a.state + static_cast<long long>(s) * a.C * HW;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  const long long n4 = HW >> 2;
  const int lane = threadIdx.x & 31;
  float vmax = 0.0f;
  int nch = 0;
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q - lane < n4;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool valid = q < n4;
    uint32_t ch = 0;  // bit j: pixel p0+j changed
    if (valid) {
      const long long p0 = q << 2;
      float4 xv[4], sv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c < a.C) {
          xv[c] = ldg_nc_f4(x + c * HW + p0);
          if (!boot) sv[c] = *reinterpret_cast<const float4*>(st + c * HW + p0);
        }
      }
      if (!boot) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < a.C) {
            ch |= static_cast<uint32_t>(fabsf(xv[c].x - sv[c].x) > tau) << 0;
            ch |= static_cast<uint32_t>(fabsf(xv[c].y - sv[c].y) > tau) << 1;
            ch |= static_cast<uint32_t>(fabsf(xv[c].z - sv[c].z) > tau) << 2;
            ch |= static_cast<uint32_t>(fabsf(xv[c].w - sv[c].w) > tau) << 3;
          }
        }
      }
      if (write_all || ch) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < a.C) {
            float4 v = xv[c];
            if (!write_all) {  // keep unchanged pixels' state (same bits written back)
              if (!(ch & 1u)) v.x = sv[c].x;
              if (!(ch & 2u)) v.y = sv[c].y;
              if (!(ch & 4u)) v.z = sv[c].z;
              if (!(ch & 8u)) v.w = sv[c].w;
            }
            *reinterpret_cast<float4*>(st + c * HW + p0) = v;
            vmax = fmaxf(vmax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
          }
        }
      }
    }
    put_quad(m, q, valid, ch, a.W, a.map_plain);
    nch += __popc(ch);
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// scalar fallback (any C, any HW): CHW state, one thread per pixel
__global__ void __launch_bounds__(kThreads) detect_frame_chw_scalar_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const float* x = *a.x_slot + static_cast<long long>(s) * a.x_sstride;
  float* st = a.state + static_cast<long long>(s) * a.C * HW;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  float vmax = 0.0f;
  int nch = 0;
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < HW;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    bool changed = false;
    if (!boot)
      for (int c = 0; c < a.C; ++c) changed |= fabsf(__ldg(x + c * HW + p) - st[c * HW + p]) > tau;
    if (changed || write_all)
      for (int c = 0; c < a.C; ++c) {
        const float v = __ldg(x + c * HW + p);
        st[c * HW + p] = v;
        vmax = fmaxf(vmax, fabsf(v));
      }
    if (changed) {
      map_set(m, p, a.W);
      ++nch;
    }
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// ---------------------------------------------------------------------------
// detect on 8-bit frames in PNM payload order ([H][W][C] interleaved bytes),
// converted as load_pnm does (io.cpp:389-397): x = float(byte) / 255.0f with
// IEEE division. One thread = 4 consecutive pixels = C 32-bit words of the
// frame; the state is CHW planes (state_chw) or NHWC (Cs == 4). C <= 4.
// ---------------------------------------------------------------------------
constexpr float kInv255 = 1.0f / 255.0f;  // fp32(1/255)
// kC: channel count known at compile time (3 = RGB PNM, the common case; 0 =
// runtime a.C <= 4). <= 64 registers: 8 CTAs per SM keep enough loads in flight.
CBG_DEV float byte_to_unit(uint32_t word, int b) {
  // load_pnm's byte / 255.0f: float(byte) via the 2^23 magic, then
  // q = byte * fp32(1/255) and one FMA residual step, which is the
  // correctly rounded quotient for all 256 bytes
  // (tests/test_ingest_math.py::test_byte_div255_sequence)
  const float fv = __uint_as_float(__byte_perm(word, 0x4B000000u, (b & 3) | 0x7540u)) - 8388608.0f;
  const float q = __fmul_rn(fv, kInv255);
  return fmaf(fmaf(-q, 255.0f, fv), kInv255, q);
}
template <bool kChw, int kC>
__global__ void __launch_bounds__(kFrameThreads, 8) detect_frame_u8_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  constexpr int CM = kC ? kC : 4;  // register arrays
  const int s = blockIdx.y;
  const int CC = kC ? kC : a.C;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const uint8_t* x8 = *a.x8_slot + static_cast<long long>(s) * CC * HW;
  float* st = a.state + static_cast<long long>(s) * (kChw ? CC : a.Cs) * HW;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  uint8_t* s8 = a.state8 ? a.state8 + static_cast<long long>(s) * CC * HW : nullptr;
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  const long long n4 = HW >> 2;
  const int lane = threadIdx.x & 31;
  float vmax = 0.0f;
  int nch = 0;
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q - lane < n4;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool valid = q < n4;
    uint32_t ch = 0;
    if (valid) {
      const long long p0 = q << 2;
      // 4 pixels x C bytes = C words, 4-byte aligned (byte offset 4*C*q)
      uint32_t wd[CM];
      const uint32_t* src = reinterpret_cast<const uint32_t*>(x8 + p0 * CC);
#pragma unroll
      for (int i = 0; i < CM; ++i) wd[i] = i < CC ? __ldg(src + i) : 0u;
      float px[4][CM];  // [pixel][channel]
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < CM; ++c) {
          if (c < CC) {
            const int b = j * CC + c;  // byte index within the 4-pixel group
            px[j][c] = byte_to_unit(wd[b >> 2], b);
          } else {
            px[j][c] = 0.0f;
          }
        }
      float sv[4][CM];
      if (!boot) {
        if constexpr (kChw) {
#pragma unroll
          for (int c = 0; c < CM; ++c)
            if (c < CC) {
              const float4 v = *reinterpret_cast<const float4*>(st + c * HW + p0);
              sv[0][c] = v.x, sv[1][c] = v.y, sv[2][c] = v.z, sv[3][c] = v.w;
            }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(st + (p0 + j) * 4);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < CM; ++c) sv[j][c] = vv[c];
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int c = 0; c < CM; ++c)
            if (c < CC && fabsf(px[j][c] - sv[j][c]) > tau) ch |= 1u << j;
      }
      if (write_all || ch) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (write_all || ((ch >> j) & 1u))
#pragma unroll
            for (int c = 0; c < CM; ++c) vmax = fmaxf(vmax, px[j][c]);
        if constexpr (kChw) {
#pragma unroll
          for (int c = 0; c < CM; ++c) {
            if (c < CC) {
              float v[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) v[j] = (write_all || ((ch >> j) & 1u)) ? px[j][c] : sv[j][c];
              *reinterpret_cast<float4*>(st + c * HW + p0) = make_float4(v[0], v[1], v[2], v[3]);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (write_all || ((ch >> j) & 1u))
              *reinterpret_cast<float4*>(st + (p0 + j) * 4) = make_float4(px[j][0], CM > 1 ? px[j][1 % CM] : 0.f, CM > 2 ? px[j][2 % CM] : 0.f, CM > 3 ? px[j][3 % CM] : 0.f);
        }
      }
      // the 8-bit shadow takes the frame's words on a full update; this kernel
      // does not track it at changed pixels, so it is valid again only after the
      // stream's next full update (detect_frame_s8_kernel keeps it current)
      if (s8 && write_all) {
        uint32_t* sdst = reinterpret_cast<uint32_t*>(s8 + p0 * CC);
#pragma unroll
        for (int i = 0; i < CM; ++i)
          if (i < CC) sdst[i] = wd[i];
      }
    }
    put_quad(m, q, valid, ch, a.W, a.map_plain);
    nch += __popc(ch);
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// The 8-bit shadow path on its own (3 channels, CHW fp32 state): everything it
// reads is bytes (12 B of frame + 12 B of shadow per 4 pixels), so each thread
// batches kQ quads, a grid stride apart, with all their loads issued first.
template <int kQ, bool kPlain>
__global__ void __launch_bounds__(kFrameThreads, 8) detect_frame_s8_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const uint8_t* x8 = *a.x8_slot + static_cast<long long>(s) * 3 * HW;
  uint8_t* s8 = a.state8 + static_cast<long long>(s) * 3 * HW;
  float* st = a.state + static_cast<long long>(s) * 3 * HW;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  const long long n4 = HW >> 2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_stream_policy();
  float vmax = 0.0f;
  int nch = 0;
  for (long long q0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q0 - lane < n4;
       q0 += kQ * stride) {
    uint32_t wd[kQ][3], sw[kQ][3];
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const long long q = q0 + u * stride;
      if (q < n4) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(x8 + 12 * q);
        const uint32_t* ssrc = reinterpret_cast<const uint32_t*>(s8 + 12 * q);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          wd[u][i] = ldg_stream_u32(src + i, pol);
          sw[u][i] = boot ? 0u : ssrc[i];
        }
      }
    }
    uint32_t chq[kQ];
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const long long q = q0 + u * stride;
      const bool valid = q < n4;
      uint32_t ch = 0;
      // a quad whose 12 bytes equal the shadow cannot change (|x - s| = 0 <= tau):
      // the common case skips the per-byte comparisons
      if (valid && !boot) {
        const bool same = (wd[u][0] == sw[u][0]) & (wd[u][1] == sw[u][1]) & (wd[u][2] == sw[u][2]);
        if (!same || tau < 0.0f) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            bool cj = false;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const int b = 3 * j + c;
              cj |= fabsf(byte_to_unit(wd[u][b >> 2], b) - byte_to_unit(sw[u][b >> 2], b)) > tau;
            }
            ch |= static_cast<uint32_t>(cj) << j;
          }
        }
      }
      if (valid && (write_all || ch)) {
        const long long p0 = q << 2;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int b = 3 * j + c;
            const bool take = write_all || ((ch >> j) & 1u);
            v[j] = byte_to_unit(take ? wd[u][b >> 2] : sw[u][b >> 2], b);
            if (take) vmax = fmaxf(vmax, v[j]);
          }
          *reinterpret_cast<float4*>(st + c * HW + p0) = make_float4(v[0], v[1], v[2], v[3]);
        }
        uint32_t* sdst = reinterpret_cast<uint32_t*>(s8 + 12 * q);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          uint32_t keep = 0;  // bytes of unchanged pixels keep the old state
          if (!write_all)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (!((ch >> ((4 * i + k) / 3)) & 1u)) keep |= 0xFFu << (8 * k);
          sdst[i] = (wd[u][i] & ~keep) | (sw[u][i] & keep);
        }
      }
      chq[u] = valid ? ch : 0u;
      nch += __popc(ch);
    }
    // map bits of the kQ groups: one vote for all of them (put_quad)
    uint32_t any = 0;
#pragma unroll
    for (int u = 0; u < kQ; ++u) any |= chq[u];
    if (__any_sync(0xffffffffu, any != 0u)) {
#pragma unroll
      for (int u = 0; u < kQ; ++u) {
        const long long q = q0 + u * stride;
        if constexpr (kPlain) {
          uint32_t v = chq[u] << (4 * (threadIdx.x & 7));
          v |= __shfl_xor_sync(0xffffffffu, v, 1);
          v |= __shfl_xor_sync(0xffffffffu, v, 2);
          v |= __shfl_xor_sync(0xffffffffu, v, 4);
          if (v && (threadIdx.x & 7) == 0) m[q >> 3] = v;  // (v != 0 only for valid groups)
        } else {
          for (int j = 0; j < 4; ++j)
            if ((chq[u] >> j) & 1u) map_set(m, (q << 2) + j, a.W);
        }
      }
    }
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// scalar fallback for 8-bit frames (HW % 4 != 0)
__global__ void __launch_bounds__(kThreads) detect_frame_u8_scalar_kernel(DetectFrameArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const uint8_t* x8 = *a.x8_slot + static_cast<long long>(s) * a.C * HW;
  const bool chw = a.state_chw != 0;
  float* st = a.state + static_cast<long long>(s) * (chw ? a.C : a.Cs) * HW;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  float vmax = 0.0f;
  int nch = 0;
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < HW;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    auto sidx = [&](int c) { return chw ? c * HW + p : p * a.Cs + c; };
    bool changed = false;
    if (!boot)
      for (int c = 0; c < a.C; ++c)
        changed |= fabsf(__fdiv_rn(static_cast<float>(x8[p * a.C + c]), 255.0f) - st[sidx(c)]) > tau;
    if (changed || write_all)
      for (int c = 0; c < a.C; ++c) {
        const float v = __fdiv_rn(static_cast<float>(x8[p * a.C + c]), 255.0f);
        st[sidx(c)] = v;
        vmax = fmaxf(vmax, v);
      }
    if (changed) {
      map_set(m, p, a.W);
      ++nch;
    }
  }
  warp_amax(a.amax ? a.amax + s : nullptr, vmax);
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// ---------------------------------------------------------------------------
// detect on NHWC inputs. A group of g lanes handles one pixel (g float4 per
// step); the group's verdict is reduced with a warp ballot.
// ---------------------------------------------------------------------------
// kCache = float4 of x each lane keeps in registers for the state write
// (ceil(Cs/4 / g), 1, 2 or 4; wider pixels re-read the rest)
template <int kCache>
__global__ void __launch_bounds__(kFrameThreads) detect_list_kernel(DetectListArgs a, int glog) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const uint32_t fno = *a.frame;
  const bool boot = a.boot[s] != 0;
  // pre-split copy: if the GEMM's exponent moved since the copy was split,
  // this frame rewrites the whole copy (dense walk; dense detection gives the
  // sparse walk's result)
  const bool has_split = a.split != nullptr;
  int e_now = 0;
  bool resplit = false;
  if (has_split) {
    e_now = f16_scale_exp(__ldg(a.amax_in + s));
    const uint32_t par = fno & 1u;
    resplit = a.split_e[(par ^ 1u) * a.S + s] != e_now;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.split_e[par * a.S + s] = e_now;
  }
  const float xs = exp2i(-e_now);
  const unsigned long long xs2 = pack_f32x2(xs, xs);
  auto put_split = [&](long long off, float4 v) {  // off: element offset of the 4-channel chunk
    uint4 w;
    f16_split2(v.x, v.y, xs2, w.x, w.z);
    f16_split2(v.z, v.w, xs2, w.y, w.w);
    *reinterpret_cast<uint4*>(a.split + off) = w;
  };
  const bool dense = boot || resplit || a.prod_idx == nullptr || (a.dense != nullptr && *a.dense != 0);
  const long long HW = static_cast<long long>(a.H) * a.W;
  const long long n = dense ? HW : a.prod_count[s * a.cnt_stride];
  const float* x = a.x + static_cast<long long>(s) * HW * a.Cs;
  float* st = a.state + static_cast<long long>(s) * HW * a.Cs;
  uint32_t* m = a.map + static_cast<long long>(s) * a.H * map_words(a.W);
  const int32_t* list = dense ? nullptr : a.prod_idx + static_cast<long long>(s) * HW;

  const int g = 1 << glog;
  const int lane = threadIdx.x & 31;
  const int sub = lane & (g - 1);
  const int gpw = 32 >> glog;                 // groups per warp
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int nv = a.Cs >> 2;                   // float4 per pixel
  const unsigned gmask = (g == 32 ? 0xffffffffu : ((1u << g) - 1u)) << ((lane >> glog) * g);
  const bool write_all = boot || !a.closed_loop;
  const float tau = a.tau[s];
  const uint64_t pol = l2_stream_policy();
  int nch = 0;

  const long long step = static_cast<long long>(gridDim.x) * wpb * gpw;
  const long long base0 = (static_cast<long long>(blockIdx.x) * wpb + warp) * gpw;
  // the next iteration's list entry is loaded one iteration ahead, so the
  // list -> data dependency costs one memory latency per warp, not one per pixel
  int p_next = (list && base0 + (lane >> glog) < n) ? __ldg(list + base0 + (lane >> glog)) : 0;
  for (long long base = base0; base < n; base += step) {
    const long long k = base + (lane >> glog);
    const bool active = k < n;
    long long p = 0;
    if (list) {
      p = p_next;
      if (k + step < n) p_next = __ldg(list + k + step);
    } else {
      p = k;
    }
    const float* xp = x + p * a.Cs;
    float* sp = st + p * a.Cs;
    // up to kCache float4 of x per lane stay in registers for the state write;
    // all loads are issued before the comparisons
    float4 xc[kCache];
    bool changed = false;
    if (active) {
      float4 sc[kCache];
#pragma unroll
      for (int j = 0; j < kCache; ++j) {
        const int v = sub + j * g;
        if (v < nv) {
          xc[j] = ldg_stream_f4(xp + 4 * v, pol);
          if (!boot) sc[j] = *reinterpret_cast<const float4*>(sp + 4 * v);
        }
      }
      if (!boot) {
#pragma unroll
        for (int j = 0; j < kCache; ++j) {
          if (sub + j * g < nv) {
            changed |= fabsf(xc[j].x - sc[j].x) > tau;
            changed |= fabsf(xc[j].y - sc[j].y) > tau;
            changed |= fabsf(xc[j].z - sc[j].z) > tau;
            changed |= fabsf(xc[j].w - sc[j].w) > tau;
          }
        }
        for (int v = sub + kCache * g; v < nv; v += g) {  // wide pixels beyond the cache
          const float4 xv = ldg_stream_f4(xp + 4 * v, pol);
          const float4 sv = *reinterpret_cast<const float4*>(sp + 4 * v);
          changed |= fabsf(xv.x - sv.x) > tau;
          changed |= fabsf(xv.y - sv.y) > tau;
          changed |= fabsf(xv.z - sv.z) > tau;
          changed |= fabsf(xv.w - sv.w) > tau;
        }
      }
    }
    const bool any = (__ballot_sync(0xffffffffu, changed) & gmask) != 0;
    if (active && (any || write_all)) {
#pragma unroll
      for (int j = 0; j < kCache; ++j)
        if (sub + j * g < nv) {
          *reinterpret_cast<float4*>(sp + 4 * (sub + j * g)) = xc[j];
          if (has_split) put_split(static_cast<long long>(s) * HW * a.Cs + p * a.Cs + 4 * (sub + j * g), xc[j]);
        }
      for (int v = sub + kCache * g; v < nv; v += g) {
        const float4 xv = ldg_nc_f4(xp + 4 * v);
        *reinterpret_cast<float4*>(sp + 4 * v) = xv;
        if (has_split) put_split(static_cast<long long>(s) * HW * a.Cs + p * a.Cs + 4 * v, xv);
      }
    } else if (active && resplit) {  // unchanged pixel, new exponent: split the kept state
      for (int v = sub; v < nv; v += g)
        put_split(static_cast<long long>(s) * HW * a.Cs + p * a.Cs + 4 * v, *reinterpret_cast<const float4*>(sp + 4 * v));
    }
    if (active && any && !boot && sub == 0) {
      map_set(m, p, a.W);
      ++nch;
    }
  }
  detect_count(a.det_count ? a.det_count + s * a.cnt_stride : nullptr, nch, boot, HW);
}

// ---------------------------------------------------------------------------
// dilate + compact on bitmaps: one warp per band of output rows.
// ---------------------------------------------------------------------------
// 32 bits of a bit-row starting at bit position B (bits outside [0, 32*nw) are 0).
CBG_DEV uint32_t bits_at(const uint32_t* row, int nw, int B) {
  const int w = B >> 5, o = B & 31;  // arithmetic shift: floor for negative B
  const uint32_t lo = (w >= 0 && w < nw) ? __ldg(row + w) : 0u;
  if (o == 0) return lo;
  const uint32_t hi = (w + 1 >= 0 && w + 1 < nw) ? __ldg(row + w + 1) : 0u;
  return __funnelshift_r(lo, hi, o);
}

// even bits of a 64-bit value (hi:lo) compacted into 32 bits
CBG_DEV uint32_t even_bits(uint32_t lo, uint32_t hi) {
  auto squeeze = [](uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
  };
  return squeeze(lo) | (squeeze(hi) << 16);
}

CBG_DEV uint32_t row_mask(int W, int wo) {  // valid bits of word wo of a W-pixel row
  const int v = W - wo * 32;
  return v >= 32 ? 0xffffffffu : (v <= 0 ? 0u : ((1u << v) - 1u));
}

// Store the words of one warp (word i of the band's map, whose bit 0 is pixel
// `pix` of the image) and append their marked pixels to the list: one atomicAdd on the stream's count per warp places the
// warp's run (row-major); a nonzero word's pixels are written by the lanes of
// its bits (coalesced). Every lane of the warp must call it (v = 0 for lanes
// without a word).
CBG_DEV void emit_words(uint32_t v, bool valid, int i, int pix, uint32_t* gmap, int32_t* list, int32_t* ctr) {
  const int lane = threadIdx.x & 31;
  if (valid) gmap[i] = v;
  const int cnt = __reduce_add_sync(0xffffffffu, __popc(v));
  if (cnt == 0) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(ctr, cnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  const uint32_t below = (1u << lane) - 1u;
  uint32_t nz = __ballot_sync(0xffffffffu, v != 0u);
  // per nonzero word: its bits and first pixel from its lane (the loop body
  // is the kernel's longest serial chain: no index arithmetic in it)
  int32_t* out = list + base;
  while (nz) {
    const int k = __ffs(nz) - 1;
    nz &= nz - 1;
    const uint32_t wk = __shfl_sync(0xffffffffu, v, k);
    const int pk = __shfl_sync(0xffffffffu, pix, k);
    const int at = __popc(wk & below);
    if ((wk >> lane) & 1u) out[at] = pk + lane;
    out += __popc(wk);
  }
}

// CTA = band of `rows` output rows of one stream, one thread per output word:
// OR the window's source words over its input rows (vertical), then dilate
// the OR-ed row horizontally with funnel shifts (stride 2 compacts the even
// bits); the loads are independent and mostly L1 hits (neighbouring words and
// rows share them). Pinned (cropped) output dims and border clipping follow
// dilate_window's bounds (change.cpp:45-61). With a fused pool, the band's
// words go to shared memory and the pool's rows inside the band (ORs of row
// pairs and bit pairs) are emitted after one barrier.
__global__ void __launch_bounds__(512) dilate_compact_kernel(DilateCompactArgs a) {
  CBG_PDL_ENTRY;
  extern __shared__ __align__(16) uint32_t s_out[];  // [rows][nwo], fused pool only
  const int s = blockIdx.y, band = blockIdx.x;
  const int nwi = (a.Win + 31) >> 5, nwo = (a.Wout + 31) >> 5;
  const bool boot = a.boot[s] != 0;
  const int r0 = band * a.rows;
  const int r1 = min(r0 + a.rows, a.Hout);
  const int nout = (r1 - r0) * nwo;
  // identity window (1x1, stride 1, same size: joins, 1x1 convs): OR of the input words
  const bool ident = a.kh == 1 && a.kw == 1 && a.stride == 1 && a.pad == 0 && a.Hin == a.Hout && a.Win == a.Wout;
  const long long in_off = static_cast<long long>(s) * a.Hin * nwi;
  const uint32_t* in_s = a.in_map[0] + in_off;
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  uint32_t* gmap = a.out_map + (static_cast<long long>(s) * a.Hout + r0) * nwo;
  for (int i0 = 0; i0 < nout; i0 += blockDim.x) {  // block-uniform
    const int i = i0 + threadIdx.x;
    const bool mine = i < nout;
    uint32_t v = 0;
    int pix = 0;
    if (mine) {
      const int rr = i / nwo, wo = i - rr * nwo;
      pix = (r0 + rr) * a.Wout + wo * 32;
      // the map loads do not wait for the boot flag's load (a boot frame
      // overrides the word at the end)
      if (a.up > 1) {  // nearest upsampling: out (jo, io) <- in (jo / up, io / up)
        const uint32_t* row = in_s + static_cast<long long>((r0 + rr) / a.up) * nwi;
        if (a.up == 2) {  // the 16 source bits of the word, each doubled
          uint32_t x = (__ldg(row + (wo >> 1)) >> (16 * (wo & 1))) & 0xFFFFu;
          x = (x | (x << 8)) & 0x00FF00FFu;
          x = (x | (x << 4)) & 0x0F0F0F0Fu;
          x = (x | (x << 2)) & 0x33333333u;
          x = (x | (x << 1)) & 0x55555555u;
          v = x | (x << 1);
        } else {
          for (int b = 0; b < 32; ++b) {
            const int c = (wo * 32 + b) / a.up;
            if (c < a.Win) v |= ((__ldg(row + (c >> 5)) >> (c & 31)) & 1u) << b;
          }
        }
        v &= row_mask(a.Wout, wo);
      } else if (ident) {
        const long long off = in_off + static_cast<long long>(r0 + rr) * nwi + wo;
        for (int q = 0; q < a.n_in; ++q) v |= __ldg(a.in_map[q] + off);
      } else {
        const int jo = r0 + rr;
        const int ja = max(jo * a.stride - a.pad, 0), jb = min(jo * a.stride - a.pad + a.kh, a.Hin);
        if (a.stride <= 2 && a.kw <= 33) {
          // the window's source bits lie in 3 (stride 1) or 4 (stride 2) consecutive words
          const int B0 = wo * 32 * a.stride - a.pad, w0 = B0 >> 5, o0 = B0 & 31;
          uint32_t x[4] = {0u, 0u, 0u, 0u};
          bool ok[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) ok[k] = w0 + k >= 0 && w0 + k < nwi && (k < 3 || a.stride == 2);
          for (int jj = ja; jj < jb; ++jj) {
            const uint32_t* row = in_s + static_cast<long long>(jj) * nwi + w0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (ok[k]) x[k] |= __ldg(row + k);
          }
          auto win = [&](int b) -> uint32_t {  // 32 bits from bit b of x[0..3]
            return b < 32 ? __funnelshift_r(x[0], x[1], b)
                          : (b < 64 ? __funnelshift_r(x[1], x[2], b - 32) : __funnelshift_r(x[2], x[3], b - 64));
          };
          if (a.stride == 1) {
            for (int ki = 0; ki < a.kw; ++ki) v |= win(o0 + ki);
          } else {
            uint32_t lo = 0, hi = 0;
            for (int ki = 0; ki < a.kw; ++ki) {
              lo |= win(o0 + ki);
              hi |= win(o0 + 32 + ki);
            }
            v = even_bits(lo, hi);
          }
        } else {
          for (int jj = ja; jj < jb; ++jj) {
            const uint32_t* row = in_s + static_cast<long long>(jj) * nwi;
            if (a.stride == 1) {
              for (int ki = 0; ki < a.kw; ++ki) v |= bits_at(row, nwi, wo * 32 - a.pad + ki);
            } else if (a.stride == 2) {
              uint32_t lo = 0, hi = 0;
              const int B0 = wo * 64 - a.pad;
              for (int ki = 0; ki < a.kw; ++ki) {
                lo |= bits_at(row, nwi, B0 + ki);
                hi |= bits_at(row, nwi, B0 + 32 + ki);
              }
              v |= even_bits(lo, hi);
            } else {
              for (int b = 0; b < 32; ++b) {
                const int io = wo * 32 + b;
                bool hit = false;
                for (int ki = 0; ki < a.kw && !hit; ++ki) {
                  const int c = io * a.stride - a.pad + ki;
                  hit = c >= 0 && c < a.Win && ((__ldg(row + (c >> 5)) >> (c & 31)) & 1u);
                }
                v |= static_cast<uint32_t>(hit) << b;
              }
            }
          }
        }
        v &= row_mask(a.Wout, wo);
      }
      if (boot) v = row_mask(a.Wout, wo);
      if (a.pool_map) s_out[i] = v;
    }
    emit_words(v, mine, i, pix, gmap, a.idx + s * HWo, a.count + s * a.cnt_stride);
  }
  if (a.pool_map == nullptr) return;
  __syncthreads();
  // fused 2x2 / stride-2 pool: pooled row pr covers band rows 2pr, 2pr+1 (the
  // second clipped at Hout), pooled bit j covers bits 2j, 2j+1
  const int nwp = (a.Wp + 31) >> 5;
  const int pr0 = r0 >> 1, pr1 = min((r1 + 1) >> 1, a.Hp);
  const int np = max(0, pr1 - pr0) * nwp;
  const int nrows = r1 - r0;
  uint32_t* pmap = a.pool_map + (static_cast<long long>(s) * a.Hp + pr0) * nwp;
  int32_t* plist = a.pool_idx + static_cast<long long>(s) * a.Hp * a.Wp;
  for (int i0 = 0; i0 < np; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool mine = i < np;
    uint32_t v = 0;
    int pix = 0;
    if (mine) {
      const int pr = i / nwp, pw = i - pr * nwp;
      pix = (pr0 + pr) * a.Wp + pw * 32;
      const int ra = 2 * (pr0 + pr) - r0, rb = ra + 1;
      auto word = [&](int r, int w) { return (r < nrows && w < nwo) ? s_out[r * nwo + w] : 0u; };
      const uint32_t lo = word(ra, 2 * pw) | word(rb, 2 * pw);
      const uint32_t hi = word(ra, 2 * pw + 1) | word(rb, 2 * pw + 1);
      v = even_bits(lo | (lo >> 1), hi | (hi >> 1)) & row_mask(a.Wp, pw);
    }
    emit_words(v, mine, i, pix, pmap, plist, a.pool_count + s * a.cnt_stride);
  }
}

// ---------------------------------------------------------------------------
// CB max-pool at listed output pixels. std::max semantics: m = (m < v) ? v : m.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ref_max(float m, float v) { return (m < v) ? v : m; }

__global__ void __launch_bounds__(kFrameThreads) pool_kernel(PoolArgs a, int glog) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const long long n = a.count[s * a.cnt_stride];
  const long long HWi = static_cast<long long>(a.Hin) * a.Win;
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  const float* x = a.x + s * HWi * a.Cs;
  float* y = a.out + s * HWo * a.Cs;
  const int32_t* list = a.idx + s * HWo;
  const int g = 1 << glog;
  const int sub = threadIdx.x & (g - 1);
  const long long gid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> glog;
  const long long gstride = (static_cast<long long>(gridDim.x) * blockDim.x) >> glog;
  const uint64_t pol = l2_stream_policy();
  const int nv = a.Cs >> 2;
  for (long long k = gid; k < n; k += gstride) {
    const int p = list[k];
    const int jo = p / a.Wout, io = p - jo * a.Wout;
    const int j0 = jo * a.stride, i0 = io * a.stride;
    const int j1 = min(j0 + a.size, a.Hin), i1 = min(i0 + a.size, a.Win);
    if (j1 - j0 == 2 && i1 - i0 == 2) {  // full 2x2 window: the four loads in flight together
      const float* q0 = x + (static_cast<long long>(j0) * a.Win + i0) * a.Cs;
      const float* q1 = q0 + static_cast<long long>(a.Win) * a.Cs;
      for (int v = sub; v < nv; v += g) {
        const float4 u00 = ldg_stream_f4(q0 + 4 * v, pol), u01 = ldg_stream_f4(q0 + a.Cs + 4 * v, pol);
        const float4 u10 = ldg_stream_f4(q1 + 4 * v, pol), u11 = ldg_stream_f4(q1 + a.Cs + 4 * v, pol);
        float4 m = u00;  // the reference's order: start at (j0, i0), then the window row-major
        const float4* us[4] = {&u00, &u01, &u10, &u11};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          m.x = ref_max(m.x, us[t]->x);
          m.y = ref_max(m.y, us[t]->y);
          m.z = ref_max(m.z, us[t]->z);
          m.w = ref_max(m.w, us[t]->w);
        }
        *reinterpret_cast<float4*>(y + static_cast<long long>(p) * a.Cs + 4 * v) = m;
      }
      continue;
    }
    for (int v = sub; v < nv; v += g) {
      float4 m = ldg_nc_f4(x + (static_cast<long long>(j0) * a.Win + i0) * a.Cs + 4 * v);
      for (int j = j0; j < j1; ++j)
        for (int i = i0; i < i1; ++i) {
          const float4 u = ldg_nc_f4(x + (static_cast<long long>(j) * a.Win + i) * a.Cs + 4 * v);
          m.x = ref_max(m.x, u.x);
          m.y = ref_max(m.y, u.y);
          m.z = ref_max(m.z, u.z);
          m.w = ref_max(m.w, u.w);
        }
      *reinterpret_cast<float4*>(y + static_cast<long long>(p) * a.Cs + 4 * v) = m;
    }
  }
}

// ---------------------------------------------------------------------------
// nearest upsampling at listed output pixels (extension): out(j, i) = in(j/f, i/f)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFrameThreads) upsample_kernel(PoolArgs a, int glog) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const long long n = a.count[s * a.cnt_stride];
  const long long HWi = static_cast<long long>(a.Hin) * a.Win;
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  const float* x = a.x + s * HWi * a.Cs;
  float* y = a.out + s * HWo * a.Cs;
  const int32_t* list = a.idx + s * HWo;
  const int g = 1 << glog;
  const int sub = threadIdx.x & (g - 1);
  const long long gid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> glog;
  const long long gstride = (static_cast<long long>(gridDim.x) * blockDim.x) >> glog;
  const int nv = a.Cs >> 2;
  for (long long k = gid; k < n; k += gstride) {
    const int p = list[k];
    const int jo = p / a.Wout, io = p - jo * a.Wout;
    const float* src = x + (static_cast<long long>(jo / a.stride) * a.Win + io / a.stride) * a.Cs;
    for (int v = sub; v < nv; v += g)
      *reinterpret_cast<float4*>(y + static_cast<long long>(p) * a.Cs + 4 * v) = ldg_nc_f4(src + 4 * v);
  }
}

// ---------------------------------------------------------------------------
// joins: one thread per (pixel, output channel).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) join_kernel(JoinArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  const long long n = a.count[s * a.cnt_stride];
  const int32_t* list = a.idx + static_cast<long long>(s) * a.HW;
  const long long total = n * a.Cs_out;
  float vmax = 0.0f;
  for (long long w = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < total;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = w / a.Cs_out;
    const int c = static_cast<int>(w - k * a.Cs_out);
    const long long p = list[k];
    float v = 0.0f;
    if (a.is_add) {
      for (int q = 0; q < a.n_in; ++q)
        v += a.in[q][(static_cast<long long>(s) * a.HW + p) * a.in_cs[q] + c];
    } else {
      int off = 0;
      for (int q = 0; q < a.n_in; ++q) {
        if (c >= off && c < off + a.in_c[q]) {
          v = a.in[q][(static_cast<long long>(s) * a.HW + p) * a.in_cs[q] + (c - off)];
          break;
        }
        off += a.in_c[q];
      }
    }
    a.out[(static_cast<long long>(s) * a.HW + p) * a.Cs_out + c] = v;
    vmax = fmaxf(vmax, fabsf(v));
  }
  warp_amax(a.amax_out ? a.amax_out + s : nullptr, vmax);
}

__global__ void begin_frame_kernel(BeginFrameArgs a) {
  if (blockIdx.x == 0) {
    const bool dense = a.dense != nullptr && *a.dense != 0;
    for (int s = threadIdx.x; s < a.S; s += blockDim.x) {
      a.boot_now[s] = static_cast<uint8_t>(a.boot_req[s] != 0 || dense);
      a.boot_req[s] = 0;
    }
    for (int i = threadIdx.x; i < a.n_nodes; i += blockDim.x) {
      a.rescan_now[i] = a.rescan_req[i];
      a.rescan_req[i] = 0;
    }
    for (int i = threadIdx.x; i < a.n_counts; i += blockDim.x)
      if (i % a.cnt_stride >= a.keep) a.counts[i] = 0;
    if (threadIdx.x == 0) {
      *a.frame += 1u;
      if (a.in_slot) *a.in_slot = a.in_ptr;
    }
  }
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n_clear;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    a.clear[i] = make_uint4(0u, 0u, 0u, 0u);
}

// ---------------------------------------------------------------------------
// delta output: pack (device -> staging, on the frame's stream); the copy-out
// stream then moves an estimated prefix [0, copied) to the host by DMA, and
// the pack itself writes any byte past that prefix straight into the mapped
// host buffer (from the SMs, only when a frame changed more than estimated)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) pack_delta_kernel(DeltaArgs a) {
  CBG_PDL_ENTRY;
  const int s = blockIdx.y;
  __shared__ size_t s_off;
  if (threadIdx.x == 0) {
    size_t off = delta_header_bytes(a.S);
    for (int j = 0; j < s; ++j) off += delta_stream_bytes(a.count[j * a.cnt_stride], a.Cs);
    s_off = off;
  }
  __syncthreads();
  const int n = a.count[s * a.cnt_stride];
  const size_t copied = static_cast<size_t>(a.copied);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    reinterpret_cast<int32_t*>(a.dst)[s] = n;
    if (4u * s >= copied) reinterpret_cast<int32_t*>(a.host)[s] = n;
  }
  const size_t ids_off = s_off, vals_off = s_off + (static_cast<size_t>(n) * 4 + 15) / 16 * 16;
  int32_t* ids = reinterpret_cast<int32_t*>(a.dst + ids_off);
  float4* vals = reinterpret_cast<float4*>(a.dst + vals_off);
  const int32_t* list = a.idx + s * a.HW;
  const int nv = a.Cs / 4;
  const float4* out = reinterpret_cast<const float4*>(a.out) + s * a.HW * nv;
  const long long total = static_cast<long long>(n) * nv;
  for (long long w = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < total;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = w / nv;
    const int v = static_cast<int>(w - k * nv);
    const int p = __ldg(list + k);
    const float4 x = ldg_nc_f4(reinterpret_cast<const float*>(out + static_cast<long long>(p) * nv + v));
    if (v == 0) {
      ids[k] = p;
      if (ids_off + 4 * k >= copied) reinterpret_cast<int32_t*>(a.host + ids_off)[k] = p;
    }
    vals[w] = x;
    if (vals_off + 16 * w >= copied) reinterpret_cast<float4*>(a.host + vals_off)[w] = x;
  }
}

__global__ void nhwc_to_chw_kernel(const float* src, float* dst, int C, int Cs, long long HW) {
  for (long long w = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < C * HW;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = w / HW, p = w - c * HW;
    dst[w] = src[p * Cs + c];
  }
}

__global__ void chw_to_nhwc_kernel(const float* src, float* dst, int C, int Cs, long long HW) {
  for (long long w = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < Cs * HW;
       w += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = w / Cs;
    const int c = static_cast<int>(w - p * Cs);
    dst[w] = c < C ? src[c * HW + p] : 0.0f;
  }
}

int group_log2(int Cs) {
  int nv = Cs / 4, glog = 0;
  while ((2 << glog) <= nv && (2 << glog) <= 32) ++glog;
  return glog;
}

}  // namespace

// The first detect merges map words in registers (no atomics) when it runs one
// of the 4-pixel kernels on rows of whole words: the same condition for both ingests.
bool detect_frame_plain_map(int C, int Cs, int W, int state_chw) {
  return W % 32 == 0 && (state_chw ? C <= 4 : Cs == 4);
}

void launch_detect_frame(const DetectFrameArgs& a, cudaStream_t st) {
  const long long HW = static_cast<long long>(a.H) * a.W;
  if (a.x8_slot) {
    if (HW % 4 == 0 && (a.state_chw || a.Cs == 4)) {
      auto go = [&](auto kernel) {
        dim3 grid(wave_grid(kernel, kFrameThreads, HW / 4, kFrameThreads, a.S, 2), a.S);
        launch_k(kernel, grid, dim3(kFrameThreads), 0, st, a);
      };
      if (a.state_chw && a.C == 3 && a.use_state8 && a.state8)
        a.map_plain ? go(detect_frame_s8_kernel<2, true>) : go(detect_frame_s8_kernel<2, false>);
      else if (a.state_chw && a.C == 3) go(detect_frame_u8_kernel<true, 3>);
      else if (a.state_chw) go(detect_frame_u8_kernel<true, 0>);
      else go(detect_frame_u8_kernel<false, 0>);
    } else {
      dim3 grid(blocks_for(HW, kThreads, a.S, sm_count()), a.S);
      launch_k(detect_frame_u8_scalar_kernel, grid, dim3(kThreads), 0, st, a);
    }
    return;
  }
  if (a.state_chw) {
    if (a.C <= 4 && HW % 4 == 0) {
      dim3 grid(wave_grid(detect_frame_chw_kernel, kFrameThreads, HW / 4, kFrameThreads, a.S, 2), a.S);
      launch_k(detect_frame_chw_kernel, grid, dim3(kFrameThreads), 0, st, a);
    } else {
      dim3 grid(blocks_for(HW, kThreads, a.S, sm_count()), a.S);
      launch_k(detect_frame_chw_scalar_kernel, grid, dim3(kThreads), 0, st, a);
    }
  } else if (a.Cs == 4 && HW % 4 == 0) {
    dim3 grid(blocks_for(HW / 4, kThreads, a.S, sm_count()), a.S);
    launch_k(detect_frame_kernel<true>, grid, dim3(kThreads), 0, st, a);
  } else {
    dim3 grid(blocks_for(HW, kThreads, a.S, sm_count()), a.S);
    launch_k(detect_frame_kernel<false>, grid, dim3(kThreads), 0, st, a);
  }
}

void launch_detect_list(const DetectListArgs& a, cudaStream_t st) {
  // lanes per pixel: two float4 of x per lane (more pixels per warp, loads in
  // flight per lane doubled) where the pixel has >= 8 of them (CBG_DETECT_PER_LANE=1: one)
  static const int per = std::getenv("CBG_DETECT_PER_LANE") ? std::max(1, std::atoi(std::getenv("CBG_DETECT_PER_LANE"))) : 2;
  int glog = group_log2(a.Cs);
  while (glog > 0 && (a.Cs / 4) / (1 << glog) < per) --glog;
  const long long HW = static_cast<long long>(a.H) * a.W;
  // 128-thread CTAs (<= 88 registers) co-reside with a persistent GEMM CTA
  const int per_lane = (a.Cs / 4 + (1 << glog) - 1) >> glog;
  auto go = [&](auto kernel) {
    dim3 grid(wave_grid(kernel, kFrameThreads, HW, kFrameThreads >> glog, a.S, 2), a.S);
    launch_k(kernel, grid, dim3(kFrameThreads), 0, st, a, glog);
  };
  if (per_lane <= 1) go(detect_list_kernel<1>);
  else if (per_lane <= 2) go(detect_list_kernel<2>);
  else go(detect_list_kernel<4>);
}

bool dilate_compact_tiling(int Hin, int Win, int Hout, int Wout, int kh, int stride, int Wp, int* rows, int* bands,
                           int* threads, int* smem_bytes) {
  (void)Hin, (void)Win, (void)kh, (void)stride;
  const int nwo = (Wout + 31) / 32;
  // ~128 output words (threads) per band (CBG_DC_THREADS; 256: 1.5 us more per
  // 64-stream frame, 512: +2.5), an even number of rows (a fused pool's rows stay inside a band)
  static const int target = std::getenv("CBG_DC_THREADS") ? std::max(32, std::atoi(std::getenv("CBG_DC_THREADS"))) : 128;
  int r = std::max(2, std::min(64, target / std::max(1, nwo))) & ~1;
  r = std::min(r, Hout + (Hout & 1));
  *rows = r;
  *bands = (Hout + r - 1) / r;
  *threads = std::min(512, ((r * nwo + 31) / 32) * 32);
  *smem_bytes = Wp > 0 ? r * nwo * 4 : 0;
  return *smem_bytes <= 48 * 1024;
}

void launch_dilate_compact(const DilateCompactArgs& a, cudaStream_t st) {
  launch_k(dilate_compact_kernel, dim3(a.n_bands, a.S), dim3(a.threads), a.pool_map ? a.smem_bytes : 0, st, a);
}

void launch_pool(const PoolArgs& a, cudaStream_t st) {
  const int glog = group_log2(a.Cs);
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  dim3 grid(wave_grid(pool_kernel, kFrameThreads, HWo, kFrameThreads >> glog, a.S, 2), a.S);
  launch_k(pool_kernel, grid, dim3(kFrameThreads), 0, st, a, glog);
}

void launch_upsample(const PoolArgs& a, cudaStream_t st) {
  const int glog = group_log2(a.Cs);
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  dim3 grid(wave_grid(upsample_kernel, kFrameThreads, HWo, kFrameThreads >> glog, a.S, 2), a.S);
  launch_k(upsample_kernel, grid, dim3(kFrameThreads), 0, st, a, glog);
}

void launch_join(const JoinArgs& a, cudaStream_t st) {
  dim3 grid(blocks_for(static_cast<long long>(a.HW) * a.Cs_out, kThreads, a.S, sm_count()), a.S);
  launch_k(join_kernel, grid, dim3(kThreads), 0, st, a);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CBG_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

const void* begin_frame_fn() { return reinterpret_cast<const void*>(&begin_frame_kernel); }

void launch_begin_frame(const BeginFrameArgs& a, cudaStream_t st) {
  const long long g = std::min<long long>(2 * sm_count(), (a.n_clear + 255) / 256);
  begin_frame_kernel<<<static_cast<int>(std::max<long long>(1, g)), 256, 0, st>>>(a);
}

void launch_pack_delta(const DeltaArgs& a, cudaStream_t st) {
  dim3 grid(std::max(1, 2 * sm_count() / std::max(1, a.S)), a.S);
  launch_k(pack_delta_kernel, grid, dim3(kThreads), 0, st, a);
}

void launch_nhwc_to_chw(const float* src, float* dst, int C, int Cs, int HW, cudaStream_t st) {
  const long long n = static_cast<long long>(C) * HW;
  nhwc_to_chw_kernel<<<static_cast<int>(std::min<long long>((n + 255) / 256, 4096)), 256, 0, st>>>(src, dst, C,
                                                                                               Cs, HW);
}

void launch_chw_to_nhwc(const float* src, float* dst, int C, int Cs, int HW, cudaStream_t st) {
  const long long n = static_cast<long long>(Cs) * HW;
  chw_to_nhwc_kernel<<<static_cast<int>(std::min<long long>((n + 255) / 256, 4096)), 256, 0, st>>>(src, dst, C,
                                                                                               Cs, HW);
}

}  // namespace cbg
