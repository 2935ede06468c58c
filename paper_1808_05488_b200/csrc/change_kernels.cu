// change_kernels.cu — HBM-bound kernels of the CBinfer hot path (sm_100a).
//
//   detect_frame    fused frame ingest (CHW) + thresholded change detection +
//                   closed-loop state update        ref change.cpp:20-43
//   detect_list     the same on NHWC inputs, walking only the producer's
//                   update set                      ref change.cpp:20-43
//   dilate_compact  window dilation of (OR-ed) change maps fused with the
//                   ordered stream compaction into the row-major index list
//                   (single pass, decoupled look-back)
//                                                   ref change.cpp:45-84
//   pool            change-based max pooling       ref layers.cpp:148-179
//   join            Add / Concat at changed pixels  ref network.cpp:364-398
//
// Arithmetic is exact IEEE fp32 (no fast-math): |x - s| > tau and the max
// comparisons are bit-identical to the reference.
#include <cstdio>

#include "common.cuh"
#include "kernels.hpp"

namespace cbg {

namespace {

constexpr int kThreads = 256;

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

// ---------------------------------------------------------------------------
// detect on the network-input frame. One thread per pixel: the C channel
// planes are read coalesced, the NHWC state as one 16-B vector per 4 channels.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) detect_frame_kernel(DetectFrameArgs a) {
  const int s = blockIdx.y;
  const uint8_t e = epoch8(*a.frame);
  const bool boot = a.boot[s] != 0;
  const long long HW = static_cast<long long>(a.H) * a.W;
  const float* x = *a.x_slot + static_cast<long long>(s) * a.C * HW;
  float* st = a.state + static_cast<long long>(s) * HW * a.Cs;
  uint8_t* m = a.map + static_cast<long long>(s) * HW;
  const bool write_all = boot || !a.closed_loop;
  const float tau = *a.tau;
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
      if (changed) m[p] = e;
    }
    if (changed || write_all) {
      for (int c0 = 0; c0 < a.Cs; c0 += 4) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (c0 + j < a.C) ? __ldg(x + (c0 + j) * HW + p) : 0.0f;
        *reinterpret_cast<float4*>(sp + c0) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// detect on NHWC inputs. A group of g lanes handles one pixel (g float4 per
// step); the group's verdict is reduced with a warp ballot.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) detect_list_kernel(DetectListArgs a, int glog) {
  const int s = blockIdx.y;
  const uint8_t e = epoch8(*a.frame);
  const bool boot = a.boot[s] != 0;
  const bool dense = boot || a.prod_idx == nullptr || (a.dense != nullptr && *a.dense != 0);
  const long long HW = static_cast<long long>(a.H) * a.W;
  const long long n = dense ? HW : a.prod_count[s];
  const float* x = a.x + static_cast<long long>(s) * HW * a.Cs;
  float* st = a.state + static_cast<long long>(s) * HW * a.Cs;
  uint8_t* m = a.map + static_cast<long long>(s) * HW;
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
  const float tau = *a.tau;

  for (long long base = (static_cast<long long>(blockIdx.x) * wpb + warp) * gpw; base < n;
       base += static_cast<long long>(gridDim.x) * wpb * gpw) {
    const long long k = base + (lane >> glog);
    const bool active = k < n;
    long long p = 0;
    if (active) p = list ? list[k] : k;
    const float* xp = x + p * a.Cs;
    float* sp = st + p * a.Cs;
    bool changed = false;
    if (active && !boot) {
      for (int v = sub; v < nv; v += g) {
        const float4 xv = ldg_nc_f4(xp + 4 * v);
        const float4 sv = *reinterpret_cast<const float4*>(sp + 4 * v);
        changed |= fabsf(xv.x - sv.x) > tau;
        changed |= fabsf(xv.y - sv.y) > tau;
        changed |= fabsf(xv.z - sv.z) > tau;
        changed |= fabsf(xv.w - sv.w) > tau;
      }
    }
    const bool any = (__ballot_sync(0xffffffffu, changed) & gmask) != 0;
    if (active && (any || write_all)) {
      for (int v = sub; v < nv; v += g)
        *reinterpret_cast<float4*>(sp + 4 * v) = ldg_nc_f4(xp + 4 * v);
    }
    if (active && any && !boot && sub == 0) m[p] = e;
  }
}

// ---------------------------------------------------------------------------
// dilate + compact. Tile = rows_per_tile output rows (<= 32 pixels/thread).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    if (lane < nw) s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == nw - 1) s_warp[32] = wi;   // block total
  }
  __syncthreads();
  total = s_warp[32];
  return s_warp[warp] + inc - v;
}

constexpr uint64_t kFlagAgg = 1ull << 30;
constexpr uint64_t kFlagInc = 2ull << 30;
constexpr uint64_t kValMask = (1ull << 30) - 1;

__global__ void __launch_bounds__(kThreads) dilate_compact_kernel(DilateCompactArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_warp[33];
  __shared__ int s_prefix;
  const int s = blockIdx.y, t = blockIdx.x;
  const uint32_t f = *a.frame;
  const uint8_t e = epoch8(f);
  const bool boot = a.boot[s] != 0;
  const int r0 = t * a.rows_per_tile;
  const int r1 = min(r0 + a.rows_per_tile, a.Hout);
  const int npix = (r1 - r0) * a.Wout;
  const long long HWin = static_cast<long long>(a.Hin) * a.Win;
  const long long HWout = static_cast<long long>(a.Hout) * a.Wout;

  const int in_lo = max(0, r0 * a.stride - a.pad);
  const int in_hi = min(a.Hin, (r1 - 1) * a.stride - a.pad + a.kh);
  const int nin = max(0, in_hi - in_lo);
  uint8_t* s_in = sm;
  uint8_t* s_h = sm + ((nin * a.Win + 15) & ~15);
  if (!boot && nin > 0) {
    for (int i = threadIdx.x; i < nin * a.Win; i += blockDim.x) {
      const long long g = static_cast<long long>(in_lo) * a.Win + i;
      uint8_t v = 0;
      for (int q = 0; q < a.n_in; ++q) v |= (a.in_map[q][s * HWin + g] == e);
      s_in[i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nin * a.Wout; i += blockDim.x) {
      const int r = i / a.Wout, io = i - r * a.Wout;
      const int c0 = io * a.stride - a.pad;
      const int ca = max(c0, 0), cb = min(c0 + a.kw, a.Win);
      uint8_t v = 0;
      for (int c = ca; c < cb; ++c) v |= s_in[r * a.Win + c];
      s_h[i] = v;
    }
    __syncthreads();
  }

  // this thread's run of consecutive tile pixels
  const int per = (npix + blockDim.x - 1) / blockDim.x;
  const int my0 = min(threadIdx.x * per, npix), my1 = min(my0 + per, npix);
  uint32_t bits = 0;
  for (int q = my0; q < my1; ++q) {
    bool set = boot;
    if (!boot && nin > 0) {
      const int jo = r0 + q / a.Wout, io = q % a.Wout;
      const int ja = max(jo * a.stride - a.pad, 0), jb = min(jo * a.stride - a.pad + a.kh, a.Hin);
      for (int jj = ja; jj < jb && !set; ++jj) set = s_h[(jj - in_lo) * a.Wout + io] != 0;
    }
    bits |= static_cast<uint32_t>(set) << (q - my0);
  }
  int agg = 0;
  const int off = block_exclusive_scan(__popc(bits), s_warp, agg);

  // decoupled look-back over the tiles of this stream
  uint64_t* stat = a.tile_status + static_cast<long long>(s) * a.n_tiles;
  const uint64_t tag = static_cast<uint64_t>(f) << 32;
  if (threadIdx.x == 0) {
    int prefix = 0;
    if (t == 0) {
      st_release_u64(&stat[0], tag | kFlagInc | static_cast<uint64_t>(agg));
    } else {
      st_release_u64(&stat[t], tag | kFlagAgg | static_cast<uint64_t>(agg));
      for (int j = t - 1; j >= 0; --j) {
        uint64_t v;
        do {
          v = ld_acquire_u64(&stat[j]);
        } while ((v >> 32) != f);
        prefix += static_cast<int>(v & kValMask);
        if ((v & kFlagInc) == kFlagInc) break;
      }
      st_release_u64(&stat[t], tag | kFlagInc | static_cast<uint64_t>(prefix + agg));
    }
    s_prefix = prefix;
    if (t == a.n_tiles - 1) a.count[s] = prefix + agg;
  }
  __syncthreads();
  int pos = s_prefix + off;
  int32_t* idx = a.idx + s * HWout;
  uint8_t* om = a.out_map + s * HWout;
  const int gbase = r0 * a.Wout;
  while (bits) {
    const int q = __ffs(bits) - 1;
    bits &= bits - 1;
    const int p = gbase + my0 + q;
    idx[pos++] = p;
    om[p] = e;
  }
}

// ---------------------------------------------------------------------------
// CB max-pool at listed output pixels. std::max semantics: m = (m < v) ? v : m.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ref_max(float m, float v) { return (m < v) ? v : m; }

__global__ void __launch_bounds__(kThreads) pool_kernel(PoolArgs a, int glog) {
  const int s = blockIdx.y;
  const long long n = a.count[s];
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
    const int j0 = jo * a.stride, i0 = io * a.stride;
    const int j1 = min(j0 + a.size, a.Hin), i1 = min(i0 + a.size, a.Win);
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
// joins: one thread per (pixel, output channel).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) join_kernel(JoinArgs a) {
  const int s = blockIdx.y;
  const long long n = a.count[s];
  const int32_t* list = a.idx + static_cast<long long>(s) * a.HW;
  const long long total = n * a.Cs_out;
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
  }
}

__global__ void begin_frame_kernel(BeginFrameArgs a) {
  const bool dense = a.dense != nullptr && *a.dense != 0;
  for (int s = threadIdx.x; s < a.S; s += blockDim.x) {
    a.boot_now[s] = static_cast<uint8_t>(a.boot_req[s] != 0 || dense);
    a.boot_req[s] = 0;
  }
  for (int i = threadIdx.x; i < a.n_nodes; i += blockDim.x) {
    a.rescan_now[i] = a.rescan_req[i];
    a.rescan_req[i] = 0;
  }
  if (threadIdx.x == 0) *a.frame += 1u;
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

void launch_detect_frame(const DetectFrameArgs& a, cudaStream_t st) {
  const long long HW = static_cast<long long>(a.H) * a.W;
  dim3 grid(blocks_for(HW, kThreads, a.S, sm_count()), a.S);
  detect_frame_kernel<<<grid, kThreads, 0, st>>>(a);
}

void launch_detect_list(const DetectListArgs& a, cudaStream_t st) {
  const int glog = group_log2(a.Cs);
  const long long HW = static_cast<long long>(a.H) * a.W;
  const int px_per_block = (kThreads >> glog);
  dim3 grid(blocks_for(HW, px_per_block, a.S, sm_count()), a.S);
  detect_list_kernel<<<grid, kThreads, 0, st>>>(a, glog);
}

int dilate_compact_smem(int Win, int Wout, int rows_per_tile, int kh, int stride) {
  const int nin = (rows_per_tile - 1) * stride + kh;
  return ((nin * Win + 15) & ~15) + nin * Wout;
}

void launch_dilate_compact(const DilateCompactArgs& a, cudaStream_t st) {
  dim3 grid(a.n_tiles, a.S);
  dilate_compact_kernel<<<grid, kThreads, a.smem_bytes, st>>>(a);
}

void launch_pool(const PoolArgs& a, cudaStream_t st) {
  const int glog = group_log2(a.Cs);
  const long long HWo = static_cast<long long>(a.Hout) * a.Wout;
  dim3 grid(blocks_for(HWo, kThreads >> glog, a.S, sm_count()), a.S);
  pool_kernel<<<grid, kThreads, 0, st>>>(a, glog);
}

void launch_join(const JoinArgs& a, cudaStream_t st) {
  dim3 grid(blocks_for(static_cast<long long>(a.HW) * a.Cs_out, kThreads, a.S, sm_count()), a.S);
  join_kernel<<<grid, kThreads, 0, st>>>(a);
}

void launch_begin_frame(const BeginFrameArgs& a, cudaStream_t st) {
  begin_frame_kernel<<<1, 256, 0, st>>>(a);
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
