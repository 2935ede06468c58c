// conv_tcgen05.cu — change-based convolution update on the 5th-gen tensor cores.
//
// Replaces, in one persistent kernel, the reference's partial im2col + GEMM +
// output update (dense.cpp:44-112, layers.cpp:10-31, layers.cpp:112-114):
//
//   for every changed output pixel p (index list and count on device)
//     Y[p, :] = act( sum_k X[p, k] * K[:, k] + bias )      scattered into
//     prev_output[p, :]  (NHWC: one contiguous Cout vector per pixel)
//
// GEMM orientation: M = changed pixels (128-row tiles), N = Cout (NPAD <= 256),
// K = kh*kw*Cs ordered (kj, ki, c) so one 16-B chunk of a K-row is one
// contiguous run of a source pixel's channel vector.
//
// Precision: 3xFP16 by default — x * 2^-e = hi + lo in fp16
// (11 + 11 significant bits, power-of-two operand scales from running magnitude
// bounds), D += Ahi*Bhi + Ahi*Blo + Alo*Bhi on tcgen05.mma kind::f16 with fp32
// accumulation in TMEM; for N <= 64 the two correction terms accumulate in
// their own TMEM columns (umma_f16x3p_kblock_ts). 3xTF32 (kind::tf32) remains
// selectable (CBG_GEMM_PREC=tf32). The same precision on the sparse and the
// dense (full-update) path.
//
// Warp roles (672 threads, 1 CTA/SM, persistent over (stream, m-tile, n-tile)):
//   epilogue (4, or 8 for N = 256): tcgen05.ld TMEM -> undo the operand scales,
//               +bias -> ReLU / leaky ReLU -> smem transpose -> 128-B stores of
//               each pixel's Cout vector
//   direct A path (default): 16 (12 for N = 256) convert warps in groups of 4,
//               one per TMEM lane quarter, each group owning every G-th K-block:
//               load the changed pixels' receptive-field chunks from global
//               memory into registers (already split by the layer's detect:
//               the pre-split copy), split if needed, tcgen05.st into the
//               stage's TMEM columns; the group leader streams the K-block's
//               pre-swizzled weight image (hi | lo) into shared memory with a
//               bulk copy on the TMA engine. A never touches shared memory.
//   staged A path (CBG_GEMM_DIRECT=0): 8 fetch warps gather the A rows with
//               16-B cp.async (zero-fill for padding taps) into swizzled smem
//               stages, completion on an mbarrier; 8 (4) convert warps split them
//               into TMEM
//   warp 20     TMEM allocator + the converged MMA issuer (elect.sync): the MMAs
//               take A from TMEM ("ts" form) and B from shared memory
// Pipelines: stages full/empty (producers <-> MMA; a stage = the B hi/lo image
// in smem + A hi/lo columns in TMEM), TMEM accumulators full/empty (MMA <->
// epilogue): two for N <= 128 so tile t's epilogue overlaps tile t+1's MMAs,
// one for N = 256 (TMEM holds 512 columns).
#include <climits>
#include <cstdio>

#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.hpp"

namespace cbg {

#ifdef CBG_TRACE
__device__ unsigned long long g_trace[6][4096];  // [event][g] clock64 of CTA 0
__device__ unsigned long long g_cta[4][160];     // per CTA: start, setup done, last MMA issued, epilogue done (ns)
__device__ unsigned long long g_epi[3][64];      // CTA 0 warp 0 per tile: saw tfull, released TMEM, stores done (clock64)
__device__ unsigned long long g_chunk[4][64];    // CTA 0 warp 0, chunks of tiles 0-7: start, TMEM landed, staged, stored
#define CHUNK_MARK(ev, c) do { if (blockIdx.x == 0 && warp == 0 && lane == 0 && (c) < 64) g_chunk[ev][c] = clock64(); } while (0)
#define EPI_MARK(ev, t) do { if (blockIdx.x == 0 && warp == 0 && lane == 0 && (t) < 64) g_epi[ev][t] = clock64(); } while (0)
CBG_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_MARK(ev) do { if (blockIdx.x < 160) g_cta[ev][blockIdx.x] = gtimer(); } while (0)
#define TRACE(ev, g) do { if (blockIdx.x == 0 && (g) < 4096) g_trace[ev][g] = clock64(); } while (0)
#else
#define TRACE(ev, g) do { } while (0)
#define CTA_MARK(ev) do { } while (0)
#define EPI_MARK(ev, t) do { } while (0)
#define CHUNK_MARK(ev, c) do { } while (0)
#endif

#ifndef CBG_GEMM_PACK
#define CBG_GEMM_PACK 1
#endif

namespace {

constexpr int kPrecTF32 = 0;
constexpr int kPrecF16 = 1;        // fp16 split, A staged through shared memory by fetch warps
constexpr int kPrecF16Direct = 2;  // fp16 split, A loaded by the convert warps straight from global
constexpr int kPrecF16Presplit = 3;  // direct, A already split by the layer's detect (ConvGemmArgs::src_presplit)
__host__ __device__ constexpr bool is_f16(int p) { return p != kPrecTF32; }
__host__ __device__ constexpr bool is_direct(int p) { return p == kPrecF16Direct || p == kPrecF16Presplit; }

// Warp roles per N tile (21 warps = 672 threads either way):
//   N <= 128: 4 epilogue, 8 fetch (2 groups), 8 convert (2 groups), 1 MMA
//   N == 256: 8 epilogue (2 per TMEM lane quarter, half the columns each: the
//             single accumulator stalls the MMAs until it is drained), 8 fetch,
//             4 convert (1 group: 128 rows of a K-block convert in ~560 cycles,
//             within the 768-cycle fp16 MMA time), 1 MMA
//   direct (kPrecF16Direct): no fetch warps; 16 (N <= 128) or 12 (N = 256)
//             convert warps in groups of 4 that load their K-block's rows from
//             global memory into registers, split them and store them into
//             TMEM with tcgen05.st.16x256b (4 threads per row, 2 rows per
//             thread per store); A never touches shared memory
// direct-path convert warps (groups of 4, one per TMEM lane quarter). Fewer
// warps free registers for the other stream groups' kernels on the GEMM's SMs
// (DESIGN.md §8.27): N = 256 runs MMA-bound with 2 groups as with 3
#ifndef CBG_N256_CONV_WARPS
#define CBG_N256_CONV_WARPS 8
#endif
#ifndef CBG_N256_EPI_WARPS  // epilogue warps of the N = 256 kernel (2 per TMEM lane quarter)
#define CBG_N256_EPI_WARPS 8
#endif
#ifndef CBG_N128_CONV_WARPS  // N <= 128
#define CBG_N128_CONV_WARPS 16
#endif
template <int NPAD, int PREC>
struct Roles {
  static constexpr int kEpiWarps = NPAD >= 256 ? CBG_N256_EPI_WARPS : 4;
  static constexpr int kFetchWarps = is_direct(PREC) ? 0 : 8;
  static constexpr int kConvWarps = is_direct(PREC) ? (NPAD >= 256 ? CBG_N256_CONV_WARPS : CBG_N128_CONV_WARPS)
                                                    : NPAD >= 256 ? 4 : 8;
  static constexpr int kFirstFetchWarp = kEpiWarps;
  static constexpr int kFirstConvWarp = kFirstFetchWarp + kFetchWarps;
  static constexpr int kMmaWarp = kFirstConvWarp + kConvWarps;
  static constexpr int kFetchGroups = 2;                   // fetch groups take alternating K-blocks
  static constexpr int kConvGroups = kConvWarps / 4;       // convert groups (128 rows each)
  static constexpr int kFetchG = is_direct(PREC) ? 128 : kFetchWarps * 32 / kFetchGroups;
  static constexpr int kConvG = 128;
  static constexpr int kFetchChunks = 128 * 8 / kFetchG;   // 16-B A chunks per fetch thread per K-block
  static constexpr int kThreads = (kMmaWarp + 1) * 32;
};
constexpr int kGroups = 2;  // stage counts are multiples of this (fetch and convert groups)
// epilogue transpose buffers: one [32][CH + 4] per epilogue warp (CH = 32, or 16 for N = 16)
__host__ __device__ constexpr int epi_buf_floats(int npad) { return (npad >= 256 ? CBG_N256_EPI_WARPS : 4) * 32 * 36; }
constexpr int kBM = 128;                 // UMMA M
constexpr int kBK = 32;                  // fp32 elements per K-block (= one 128-B swizzle row)
constexpr int kABytes = kBM * kBK * 4;   // raw fp32 A rows of one K-block: 16 KB
constexpr int kMaxS = 1024;

// Operand precision of the split-fp32 product (both fp32-accurate):
//   kPrecTF32: x = hi + lo in tf32 (hi = x truncated to 10 mantissa bits),
//              kind::tf32, K = 8 per MMA, B rows of 128 B (32 fp32) per K-block.
//   kPrecF16:  x*2^-e = hi + lo in fp16 (round-to-nearest, 11 + 11 bits), with
//              e a per-stream power-of-two scale from a running bound of the
//              operand magnitude (so |x*2^-e| < 2^15: no overflow), weights
//              scaled by 2^-ew on the host; kind::f16 at twice the tf32 rate,
//              K = 16 per MMA, B rows of 64 B (32 fp16) per K-block (SW64);
//              the epilogue multiplies by 2^(e+ew) (exact).
template <int NPAD, int PREC>
struct Cfg {
  static constexpr int kBRow = is_f16(PREC) ? 64 : 128;  // B bytes per row per K-block
  static constexpr int kBBytes = NPAD * kBRow;
  static constexpr int kStageBytes = (is_direct(PREC) ? 0 : kABytes) + 2 * kBBytes;
  static constexpr int kACols = is_f16(PREC) ? kBK : 2 * kBK;  // TMEM columns of A_hi | A_lo
  static constexpr int kALo = kACols / 2;                          // A_lo column offset
  // A multiple of kGroups, so a stage is always filled and converted by the same
  // group: with an odd count, a convert group could reach a stage one lap ahead
  // of the other group's fetch and take that stage's previous `raw` phase
  // (mbarrier parity aliases modulo 2) as complete.
  // (N = 256 has one convert group, so any count works there; 3 leaves room
  // for its 8 epilogue warps' transpose buffers)
  static constexpr int kStages = is_direct(PREC) ? (NPAD >= 256 ? (CBG_N256_CONV_WARPS == 12 ? 3 : 4)
                                                                : (CBG_N128_CONV_WARPS == 12 ? 6 : 8))
                                 : is_f16(PREC)  ? (NPAD >= 256 ? 3 : NPAD >= 128 ? 6 : 8)
                                                 : (NPAD >= 256 ? 2 : NPAD >= 128 ? 4 : 6);
  static_assert(kStages % Roles<NPAD, PREC>::kConvGroups == 0, "stages must be a multiple of the convert groups");
  static constexpr int kNAcc = NPAD >= 256 ? 1 : 2;  // TMEM accumulator buffers
  // fp16, N <= 64: a separate accumulator for the two correction terms
  // (umma_f16x3p_kblock_ts), so an accumulator buffer is [main | corr]
  static constexpr bool kPack = is_f16(PREC) && NPAD <= 64 && CBG_GEMM_PACK;
  static constexpr int kAccCols = kPack ? 2 * NPAD : NPAD;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kAColBase = kNAcc * kAccCols;  // first A stage column
  static_assert(kNAcc * kAccCols + kStages * kACols <= 512, "TMEM budget");
};

__host__ __device__ constexpr int tail_bytes(int stages, int KB, int S, int nbias, int npad, bool direct) {
  return 8 * (3 * stages + 4) + 16 + kBM * 8 + (S + 1) * 4 + 16 + 4 * epi_buf_floats(npad) + 4 * nbias +
         (direct ? 8 * 8 * KB : 0);
}

template <int NPAD, int PREC>
__global__ void __maxnreg__(80)  // 21 warps (17 for the 8-convert-warp N = 256 variant) x 80 registers
    conv_gemm_kernel(const __grid_constant__ ConvGemmArgs a) {
  using C = Cfg<NPAD, PREC>;
  using R = Roles<NPAD, PREC>;
  constexpr int kThreads = R::kThreads;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tail = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty = full + C::kStages;
  uint64_t* raw = empty + C::kStages;  // fetch -> convert (cp.async landed)
  uint64_t* tfull = raw + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int2* rowinfo = reinterpret_cast<int2*>(tmem_holder + 4);
  int* tprefix = reinterpret_cast<int*>(rowinfo + kBM);
  float* epi_buf = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(tprefix + a.S + 1) + 15) & ~uintptr_t(15));  // [4 warps][32][CH + 4]
  float* s_bias = epi_buf + epi_buf_floats(NPAD);                              // [n_tiles * NPAD]
  uint2* s_ktab = reinterpret_cast<uint2*>(s_bias + a.n_tiles * NPAD);          // direct: [KB * 8]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  pdl_trigger();
  if (tid == 0) CTA_MARK(0);
  const long long HWin = static_cast<long long>(a.Hin) * a.Win;
  const long long HWout = static_cast<long long>(a.Hout) * a.Wout;

  // ---- setup -----------------------------------------------------------------
  if (tid == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], R::kConvWarps / R::kConvGroups + 1);  // one convert group + 1 expect_tx arrive
      mbar_init(&empty[i], 1);              // tcgen05.commit
      mbar_init(&raw[i], a.use_tma ? 1 : R::kFetchG);  // one cp.async arrive per fetch thread of a group, or the TMA
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], R::kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == R::kMmaWarp) tmem_alloc(tmem_holder, C::kTmemCols);
  for (int i = tid; i < a.n_tiles * NPAD; i += kThreads) s_bias[i] = a.bias[i];  // zero-padded to n_tiles*NPAD
  if constexpr (is_direct(PREC))
    for (int i = tid; i < a.KB * 8; i += kThreads) s_ktab[i] = reinterpret_cast<const uint2*>(a.ktab)[i];
  pdl_wait();  // the setup above (barriers, TMEM, bias, tap table) does not read the predecessor's results
  if (warp == 0) {
    int carry = 0;
    if (lane == 0) tprefix[0] = 0;
    for (int s0 = 0; s0 < a.S; s0 += 32) {
      const int s = s0 + lane;
      const int v = s < a.S ? ((a.count[s * a.cnt_stride] + kBM - 1) / kBM) * a.n_tiles : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      if (s < a.S) tprefix[s + 1] = carry + inc;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int total = tprefix[a.S];
  if (tid == 0) CTA_MARK(1);

  auto decode = [&](int w, int& s, int& mt, int& nt) {
    int lo = 0, hi = a.S;  // find s with tprefix[s] <= w < tprefix[s+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (tprefix[mid] <= w) lo = mid;
      else hi = mid;
    }
    s = lo;
    const int local = w - tprefix[s];
    mt = local / a.n_tiles;
    nt = local - mt * a.n_tiles;
  };

  if (!is_direct(PREC) && a.use_tma && warp >= R::kFirstFetchWarp && warp < R::kFirstConvWarp) {
    // ===================== fetch by TMA gather4 (1x1 layers) =====================
    // one thread per fetch group issues, per K-block, 32 gather4 copies of 4 rows
    // x 128 B (the K-block's 32 fp32 of 4 changed pixels) into the stage, 128-B
    // swizzled exactly like the cp.async path's manual XOR, completing on the
    // stage's `raw` barrier; rows past the count read an out-of-range row (zeros)
    const int wpg = R::kFetchWarps / R::kFetchGroups;
    const int fgrp = (warp - R::kFirstFetchWarp) / wpg;
    const bool lead_warp = (warp - R::kFirstFetchWarp) % wpg == 0;
    const int oob = a.S * static_cast<int>(HWin);  // first row past the tensor
    int* s_rows = reinterpret_cast<int*>(rowinfo) + fgrp * kBM;  // this group's tile rows (tensor rows)
    uint32_t g = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int s, mt, nt;
      decode(w, s, mt, nt);
      if (!lead_warp) {
        g += a.KB;
        continue;
      }
      const int cnt = a.count[s * a.cnt_stride];
      // the tile's rows -> input pixels (1x1, stride 1, pad 0; the output may be a crop)
      for (int j = lane; j < kBM; j += 32) {
        const int k = mt * kBM + j;
        int row = oob;
        if (k < cnt) {
          const int p = __ldg(a.idx + s * HWout + k);
          const int jo = p / a.Wout, io = p - jo * a.Wout;
          row = s * static_cast<int>(HWin) + jo * a.Win + io;
        }
        s_rows[j] = row;
      }
      __syncwarp();
      const uint8_t* bimg = a.wimg + static_cast<long long>(nt) * a.KB * 2 * C::kBBytes;
#pragma unroll 1
      for (int kb = 0; kb < a.KB; ++kb, ++g) {
        if (static_cast<int>(g % R::kFetchGroups) != fgrp) continue;
        const int stage = g % C::kStages;
        const uint32_t phase = (g / C::kStages) & 1;
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&raw[stage], kABytes);
        }
        __syncwarp();
        uint8_t* sA = smem + stage * C::kStageBytes;
        {  // lane i issues the gather4 of rows 4i..4i+3 (32 lanes x 4 rows = the tile)
          const int4 r = make_int4(s_rows[4 * lane], s_rows[4 * lane + 1], s_rows[4 * lane + 2], s_rows[4 * lane + 3]);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(sA + 512 * lane)),
              "l"(reinterpret_cast<uint64_t>(&a.tmap)), "r"(32 * kb), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
              "r"(smem_u32(&raw[stage]))
              : "memory");
        }
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[stage], 2 * C::kBBytes);
          bulk_g2s(sA + kABytes, bimg + static_cast<long long>(kb) * 2 * C::kBBytes, 2 * C::kBBytes, &full[stage]);
        }
      }
      __syncwarp();
    }
  } else if (warp >= R::kFirstFetchWarp && warp < R::kFirstConvWarp) {
    // ========================= fetch =========================
    constexpr int kFetchG = R::kFetchG, kFetchChunks = R::kFetchChunks;
    const int fgrp = (tid - 32 * R::kFirstFetchWarp) / kFetchG;  // K-blocks g with g % groups == fgrp
    const int ftid = (tid - 32 * R::kFirstFetchWarp) % kFetchG;
    const int q = ftid & 7;
    const uint2* ktab = reinterpret_cast<const uint2*>(a.ktab);  // (tap code, element offset) per 16-B chunk
    uint32_t g = 0;  // global K-block counter (stage = g % kStages)
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int s, mt, nt;
      decode(w, s, mt, nt);
      const int cnt = a.count[s * a.cnt_stride];
      // this thread's rows of the tile -> receptive-field origins, in registers
      int jb[kFetchChunks], ib[kFetchChunks], roff[kFetchChunks];
#pragma unroll
      for (int i = 0; i < kFetchChunks; ++i) {
        const int k = mt * kBM + i * (kFetchG / 8) + (ftid >> 3);
        const int p = k < cnt ? __ldg(a.idx + s * HWout + k) : -1;
        const int jo = p / a.Wout, io = p - jo * a.Wout;
        jb[i] = p >= 0 ? jo * a.stride - a.pad : INT_MIN / 2;
        ib[i] = io * a.stride - a.pad;
        roff[i] = (jb[i] * a.Win + ib[i]) * a.Cs;
      }
      const float* src = a.src + s * HWin * a.Cs;
      const uint8_t* bimg = a.wimg + static_cast<long long>(nt) * a.KB * 2 * C::kBBytes;
#pragma unroll 1
      for (int kb = 0; kb < a.KB; ++kb, ++g) {
        if (static_cast<int>(g % R::kFetchGroups) != fgrp) continue;
        const int stage = g % C::kStages;
        const uint32_t phase = (g / C::kStages) & 1;
        const uint2 tk = __ldg(ktab + kb * 8 + q);
        const uint32_t tab = tk.x;
        const int toff = static_cast<int>(tk.y);
        const int dj = tab & 0xFF, di = (tab >> 8) & 0xFF;
        const bool tap_ok = (tab >> 31) == 0;
        mbar_wait(&empty[stage], phase ^ 1);
        if (ftid == 0) TRACE(4, g);
        uint8_t* sA = smem + stage * C::kStageBytes;
        const uint32_t base = smem_u32(sA);
#pragma unroll
        for (int i = 0; i < kFetchChunks; ++i) {
          const int r = i * (kFetchG / 8) + (ftid >> 3);
          const bool ok = tap_ok && static_cast<unsigned>(jb[i] + dj) < static_cast<unsigned>(a.Hin) &&
                          static_cast<unsigned>(ib[i] + di) < static_cast<unsigned>(a.Win);
          cp_async16(base + r * 128 + ((q ^ (r & 7)) << 4), ok ? src + (roff[i] + toff) : src, ok ? 16u : 0u);
        }
        cp_async_mbar_arrive(&raw[stage]);
        // the weight K-block on the TMA engine, after this thread's gather copies
        // are queued (issuing it first delayed the whole warp's copies)
        if (ftid == 32) {
          mbar_arrive_expect_tx(&full[stage], 2 * C::kBBytes);
          bulk_g2s(sA + kABytes, bimg + static_cast<long long>(kb) * 2 * C::kBBytes, 2 * C::kBBytes,
                   &full[stage]);
        }
        if (ftid == 0) TRACE(0, g);
      }
    }
  } else if (is_direct(PREC) && warp >= R::kFirstConvWarp && warp < R::kMmaWarp) {
    // ===================== direct load + convert =====================
    // Group `grp` (4 warps, one per TMEM lane quarter) owns K-blocks g with
    // g % groups == grp. A thread holds chunks c and c+4 (16 B each) of rows
    // a, a+8 (+16, +24) of its quarter: exactly the register layout of
    // tcgen05.st.16x256b.x2 (lane a: cols 2c..2c+1 and 8+2c..; lane a+8: same).
    // Each load instruction reads 4 consecutive chunks (64 B) of 8 rows.
    const int grp = (warp - R::kFirstConvWarp) >> 2;
    const int quarter = warp & 3;
    const int c = lane & 3, arow = lane >> 2;
    const uint32_t ktab_s = smem_u32(s_ktab);
    const bool leader = (warp & 3) == 0 && lane == 0;  // issues the group's weight copies
    constexpr int G = R::kConvGroups;
    uint32_t g = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int s, mt, nt;
      decode(w, s, mt, nt);
      const int cnt = a.count[s * a.cnt_stride];
      const float xs = exp2i(-f16_scale_exp(__ldg(a.amax_in + s)));
      const unsigned long long xs2 = pack_f32x2(xs, xs);
      // rows (h, b) = 32*quarter + 16*h + 8*b + arow
      int jb[4], ib[4];
      const float* rowp[4];  // the row's receptive-field origin (may point before the image: offsets are added)
      const float* src = a.src + s * HWin * a.Cs;
      bool inside = true;    // all four rows valid with their whole window inside the image
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = mt * kBM + 32 * quarter + 8 * i + arow;
        // the list load does not wait for the count (rows past it are masked after)
        const int pr = __ldg(a.idx + s * HWout + min(k, static_cast<int>(HWout) - 1));
        const int p = k < cnt ? pr : -1;
        const int jo = p / a.Wout, io = p - jo * a.Wout;
        jb[i] = p >= 0 ? jo * a.stride - a.pad : INT_MIN / 2;
        ib[i] = io * a.stride - a.pad;
        rowp[i] = src + static_cast<long long>(p >= 0 ? (jb[i] * a.Win + ib[i]) * a.Cs : 0);
        inside = inside && p >= 0 && jb[i] >= 0 && jb[i] + a.kh <= a.Hin && ib[i] >= 0 && ib[i] + a.kw <= a.Win;
      }
      // warp-uniform: the whole warp takes the unchecked loads or none of it
      const bool fast = __all_sync(0xffffffffu, inside);
      const uint8_t* bimg = a.wimg + static_cast<long long>(nt) * a.KB * 2 * C::kBBytes;
      // rows 2h, 2h+1 of K-block kb -> v[2h..2h+1]
      auto load_half = [&](int kb, int h, float4 (&v)[4][2]) {
        const uint2 t0 = lds_u2(ktab_s + 8u * (kb * 8 + c)), t1 = lds_u2(ktab_s + 8u * (kb * 8 + c + 4));
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int i = 2 * h + b;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint2 tk = j ? t1 : t0;
            bool ok = (tk.x >> 31) == 0;  // K padding
            if (!fast) {
              const int dj = tk.x & 0xFF, di = (tk.x >> 8) & 0xFF;
              ok = ok && static_cast<unsigned>(jb[i] + dj) < static_cast<unsigned>(a.Hin) &&
                   static_cast<unsigned>(ib[i] + di) < static_cast<unsigned>(a.Win);
            }
            v[i][j] = ok ? ldg_nc_f4(rowp[i] + static_cast<int>(tk.y)) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      };
      const uint32_t g0 = g;  // K-block counter at the tile's start; this group's first is kb0
      const int kb0 = static_cast<int>((grp + G - g0 % G) % G);
      g = g0 + a.KB;
#pragma unroll 1
      for (int kb = kb0; kb < a.KB; kb += G) {
        const uint32_t gk = g0 + kb;
        const int stage = gk % C::kStages;
        const uint32_t phase = (gk / C::kStages) & 1;
        float4 v[4][2];
        load_half(kb, 0, v);  // loads first: they do not depend on the stage being free
        load_half(kb, 1, v);
        mbar_wait(&empty[stage], phase ^ 1);  // TMEM A stage and B smem free
        if (leader) {
          TRACE(4, gk);
          mbar_arrive_expect_tx(&full[stage], 2 * C::kBBytes);
          bulk_g2s(smem + stage * C::kStageBytes, bimg + static_cast<long long>(kb) * 2 * C::kBBytes,
                   2 * C::kBBytes, &full[stage]);
        }
        const uint32_t ta = tmem_base + (static_cast<uint32_t>(32 * quarter) << 16) + C::kAColBase +
                            stage * C::kACols;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // TMEM lanes 32q + 16h .. +15
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 2; ++j)      // chunk c, c+4 -> column pairs 2c.., 8+2c..
#pragma unroll
            for (int b = 0; b < 2; ++b) {  // row a, a+8 -> registers 0-1 / 2-3 (+4 for chunk c+4)
              const float4 x = v[2 * h + b][j];
              if constexpr (PREC == kPrecF16Presplit) {  // the detect split the chunk: {hi01, hi23, lo01, lo23}
                hi[4 * j + 2 * b] = __float_as_uint(x.x);
                hi[4 * j + 2 * b + 1] = __float_as_uint(x.y);
                lo[4 * j + 2 * b] = __float_as_uint(x.z);
                lo[4 * j + 2 * b + 1] = __float_as_uint(x.w);
              } else {
                f16_split2(x.x, x.y, xs2, hi[4 * j + 2 * b], lo[4 * j + 2 * b]);
                f16_split2(x.z, x.w, xs2, hi[4 * j + 2 * b + 1], lo[4 * j + 2 * b + 1]);
              }
            }
          tmem_st_16x256b_x2(ta + (static_cast<uint32_t>(16 * h) << 16), hi);
          tmem_st_16x256b_x2(ta + (static_cast<uint32_t>(16 * h) << 16) + C::kALo, lo);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
        if (leader) TRACE(5, gk);
      }
    }
  } else if (warp >= R::kFirstConvWarp && warp < R::kMmaWarp) {
    // ========================= convert =========================
    const int cgrp = (tid - R::kFirstConvWarp * 32) / R::kConvG;
    const int ctid = (tid - R::kFirstConvWarp * 32) % R::kConvG;
    uint32_t g = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      float xs = 1.0f;  // fp16 operand scale 2^-e of this tile's stream
      if constexpr (is_f16(PREC)) {
        int s, mt, nt;
        decode(w, s, mt, nt);
        xs = exp2i(-f16_scale_exp(__ldg(a.amax_in + s)));
      }
#pragma unroll 1
      for (int kb = 0; kb < a.KB; ++kb, ++g) {
        if (static_cast<int>(g % R::kConvGroups) != cgrp) continue;
        const int stage = g % C::kStages;
        const uint32_t phase = (g / C::kStages) & 1;
        mbar_wait(&raw[stage], phase);
        if (ctid == 0) TRACE(1, g);
        uint8_t* sA = smem + stage * C::kStageBytes;
        // thread = row r of the tile (= its TMEM lane: warp % 4 picks the lane
        // quarter a warp may access); the 8 swizzled 16-B chunks of the row
        const int r = 32 * (warp & 3) + lane;
        const uint32_t row = smem_u32(sA) + r * 128;
        const uint32_t ta = tmem_base + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + C::kAColBase +
                            stage * C::kACols;
        if constexpr (is_f16(PREC)) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {  // 16 elements -> 8 packed columns each of hi and lo
            uint32_t h[8], l[8];
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const int q = 4 * half + qq;
              float x[4];
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                           : "r"(row + ((q ^ (r & 7)) << 4)));
              // x*2^-e exact; hi = fp16 round-to-nearest, lo = fp16(x - hi)
              // (x - hi exact in fp32): hi + lo carries 22 significant bits
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const float x0 = x[2 * j] * xs, x1 = x[2 * j + 1] * xs;
                const __half2 hh = __floats2half2_rn(x0, x1);
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
                h[2 * qq + j] = *reinterpret_cast<const uint32_t*>(&hh);
                l[2 * qq + j] = *reinterpret_cast<const uint32_t*>(&ll);
              }
            }
            tmem_st8(ta + 8 * half, h);
            tmem_st8(ta + C::kALo + 8 * half, l);
          }
        } else {
#pragma unroll
          for (int half = 0; half < 2; ++half) {  // 16 columns at a time (register pressure)
            uint32_t h[16], l[16];
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const int q = 4 * half + qq;
              float x[4];
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                           : "r"(row + ((q ^ (r & 7)) << 4)));
              // hi = x truncated to tf32 (exactly representable), lo = x - hi
              // (exact in fp32); the tensor core reads lo to tf32 precision, so
              // hi + lo carries ~21 significant bits of x.
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                h[4 * qq + j] = __float_as_uint(x[j]) & 0xFFFFE000u;
                l[4 * qq + j] = __float_as_uint(x[j] - __uint_as_float(h[4 * qq + j]));
              }
            }
            tmem_st16(ta + 16 * half, h);
            tmem_st16(ta + C::kALo + 16 * half, l);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
        if (ctid == 0) TRACE(5, g);
      }
    }
  } else if (warp == R::kMmaWarp) {
    // ========================= MMA issuer =========================
    // The whole warp runs the loop (warp-uniform control flow and operands);
    // elect.sync inside the asm picks the issuing lane.
    constexpr uint32_t idesc = is_f16(PREC) ? umma_idesc_f16(kBM, NPAD) : umma_idesc_tf32(kBM, NPAD);
    constexpr uint32_t idesc2 = umma_idesc_f16(kBM, 2 * NPAD);  // packed: A_hi x [B_hi; B_lo]
    // stage 0 base; B by offset (K-major, 128-B rows for tf32, 64-B rows for fp16)
    const uint64_t desc0 = is_f16(PREC) ? umma_desc_sw64(smem_u32(smem)) : umma_desc_sw128(smem_u32(smem));
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t gm = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tbase + acc * C::kAccCols;
      for (int kb = 0; kb < a.KB; ++kb) {
        mbar_wait(&full[stage], phase);
        TRACE(2, gm);
        tc_fence_after();
        // B descriptors: start addresses advance in 16-B units; A in TMEM
        const uint64_t b_hi =
            desc0 + static_cast<uint64_t>((stage * C::kStageBytes + (is_direct(PREC) ? 0 : kABytes)) >> 4);
        const uint64_t b_lo = b_hi + (C::kBBytes >> 4);
        const uint32_t a_hi = tbase + C::kAColBase + stage * C::kACols;
        if constexpr (C::kPack)
          umma_f16x3p_kblock_ts(d, d + NPAD, a_hi, a_hi + C::kALo, b_hi, idesc2, idesc, kb != 0);
        else if constexpr (is_f16(PREC))
          umma_f16x3_kblock_ts(d, a_hi, a_hi + C::kALo, b_hi, b_lo, idesc, kb != 0);
        else
          umma_tf32x3_kblock_ts(d, a_hi, a_hi + C::kALo, b_hi, b_lo, idesc, kb != 0);
        umma_commit_elect(&empty[stage]);  // smem slot free once these MMAs retire
        TRACE(3, gm);
        ++gm;
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit_elect(&tfull[acc]);
      if (++acc == C::kNAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) CTA_MARK(2);
  } else if (warp < R::kEpiWarps) {
    // ========================= epilogue =========================
    // Per chunk of CH accumulator columns: tcgen05.ld (lane = row) -> scale,
    // bias, ReLU -> the warp's smem transpose buffer -> global stores in which
    // CH/4 consecutive lanes write one pixel's CH contiguous outputs (full
    // 32-B sectors; lane = row would scatter 32 rows per store instruction).
    constexpr int CH = (NPAD >= 32 && !C::kPack) ? 32 : 16;  // packed: two CH-column loads per chunk
    constexpr int LPR = CH / 4;     // lanes per pixel row in the store phase
    constexpr int RPI = 32 / LPR;   // pixel rows per store instruction
    constexpr int NCOL = NPAD / (R::kEpiWarps / 4);  // accumulator columns of this warp
    const int quarter = warp & 3;                     // TMEM lanes 32*quarter .. +31 (= warp % 4)
    const int col0 = (warp >> 2) * NCOL;
    const uint32_t tbuf_u32 = smem_u32(epi_buf + warp * 32 * (CH + 4));
    const uint32_t s_bias_u32 = smem_u32(s_bias);
    int acc = 0;
    uint32_t acc_phase = 0;
    int tile_no = 0;
    (void)tile_no;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int s, mt, nt;
      decode(w, s, mt, nt);
      const int cnt = a.count[s * a.cnt_stride];
      const int k = mt * kBM + quarter * 32 + lane;
      const bool valid = k < cnt;
      const int p = valid ? a.idx[s * HWout + k] : -1;
      float* obase = a.out + s * HWout * a.Co4;
      const int nbase = nt * NPAD;
      float ys = 1.0f, ws = 1.0f;  // undo the fp16 operand scales: y * 2^e * 2^ew (both exact)
      if constexpr (is_f16(PREC)) {
        ys = exp2i(f16_scale_exp(__ldg(a.amax_in + s)));
        ws = exp2i(a.w_exp);
      }
      float vmax = 0.0f;  // |written value| bound for the consumers' scales
      mbar_wait(&tfull[acc], acc_phase);
      EPI_MARK(0, tile_no);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * C::kAccCols;
#pragma unroll 1
      for (int n0 = col0; n0 < col0 + NCOL; n0 += CH) {
        const int cidx = tile_no * (NCOL / CH) + (n0 - col0) / CH;
        (void)cidx;
        CHUNK_MARK(0, cidx);
        uint32_t r[CH];
        if constexpr (CH == 32) tmem_ld32(tb + n0, r);
        else tmem_ld16(tb + n0, r);
        if constexpr (C::kPack) {  // main + correction accumulator, one fp32 add
          uint32_t r2[CH];
          tmem_ld16(tb + NPAD + n0, r2);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CH; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
        }
        tmem_ld_wait();
        CHUNK_MARK(1, cidx);
        if (n0 + CH >= col0 + NCOL) {  // this warp's last TMEM read of the tile: hand its part back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          EPI_MARK(1, tile_no);
        }
        // shared-memory traffic as explicit ld/st.shared (the buffers' generic
        // pointers compiled to generic LD/ST); no "memory" clobbers, so the
        // compiler keeps them in flight together; bar.warp.sync orders them
        const uint32_t bias_s = s_bias_u32 + 4u * static_cast<uint32_t>(nbase + n0);
        const uint32_t row_s = tbuf_u32 + 4u * static_cast<uint32_t>(lane * (CH + 4));
#pragma unroll
        for (int j = 0; j < CH / 4; ++j) {
          const float4 b = lds_f4(bias_s + 16u * j);  // broadcast
          float o[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float y = __uint_as_float(r[4 * j + u]);
            // (y * 2^e) * 2^ew + b: the products are exact, so the fused form
            // rounds once, like the reference's y + b
            if constexpr (is_f16(PREC)) y = fmaf(y * ys, ws, (&b.x)[u]);
            else y = y + (&b.x)[u];
            if (a.relu) y = (y < 0.0f) ? (a.slope != 0.0f ? y * a.slope : 0.0f) : y;  // std::max(v, 0.f) / leaky
            o[u] = y;
            vmax = fmaxf(vmax, fabsf(y));
          }
          sts_f4(row_s + 16u * j, make_float4(o[0], o[1], o[2], o[3]));
        }
        if (!valid) vmax = 0.0f;
        warp_sync_mem();
        CHUNK_MARK(2, cidx);
        const int c4 = lane % LPR;
        const int n = nbase + n0 + 4 * c4;
        float4 v[32 / RPI];
        int pr[32 / RPI];
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int rr = i * RPI + lane / LPR;
          pr[i] = __shfl_sync(0xffffffffu, p, rr);
          v[i] = lds_f4(tbuf_u32 + 4u * static_cast<uint32_t>(rr * (CH + 4) + 4 * c4));
        }
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i)
          if (pr[i] >= 0 && n < a.Co4) *reinterpret_cast<float4*>(obase + static_cast<long long>(pr[i]) * a.Co4 + n) = v[i];
        warp_sync_mem();
        CHUNK_MARK(3, cidx);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
      if (lane == 0 && a.amax_out) atomicMax(reinterpret_cast<int*>(a.amax_out + s), __float_as_int(vmax));
      EPI_MARK(2, tile_no);
      ++tile_no;
      if (++acc == C::kNAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (tid == 0) CTA_MARK(3);
  if (warp == R::kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

template <int NPAD, int PREC>
void launch_impl(const ConvGemmArgs& a, cudaStream_t st) {
  const int smem = conv_gemm_smem_bytes(NPAD, a.KB, a.S, PREC, a.n_tiles);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(conv_gemm_kernel<NPAD, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    configured = true;
  }
  launch_k(conv_gemm_kernel<NPAD, PREC>, dim3(a.grid), dim3(Roles<NPAD, PREC>::kThreads), smem, st, a);
}

template <int PREC>
void launch_prec(const ConvGemmArgs& a, cudaStream_t st) {
  switch (a.npad) {
    case 16: launch_impl<16, PREC>(a, st); break;
    case 32: launch_impl<32, PREC>(a, st); break;
    case 64: launch_impl<64, PREC>(a, st); break;
    case 128: launch_impl<128, PREC>(a, st); break;
    default: launch_impl<256, PREC>(a, st); break;
  }
}

template <int PREC>
int stages_prec(int npad) {
  switch (npad) {
    case 16: return Cfg<16, PREC>::kStages;
    case 32: return Cfg<32, PREC>::kStages;
    case 64: return Cfg<64, PREC>::kStages;
    case 128: return Cfg<128, PREC>::kStages;
    default: return Cfg<256, PREC>::kStages;
  }
}

}  // namespace

int conv_gemm_read_trace(unsigned long long* host, int n) {
#ifdef CBG_TRACE
  if (n >= 6 * 4096 + 4 * 160) {
    if (cudaMemcpyFromSymbol(host + 6 * 4096, g_cta, sizeof(unsigned long long) * 4 * 160) != cudaSuccess) return -1;
  }
  if (n >= 6 * 4096 + 4 * 160 + 3 * 64) {
    if (cudaMemcpyFromSymbol(host + 6 * 4096 + 4 * 160, g_epi, sizeof(unsigned long long) * 3 * 64) != cudaSuccess)
      return -1;
  }
  if (n >= 6 * 4096 + 4 * 160 + 7 * 64) {
    if (cudaMemcpyFromSymbol(host + 6 * 4096 + 4 * 160 + 3 * 64, g_chunk, sizeof(unsigned long long) * 4 * 64) !=
        cudaSuccess)
      return -1;
  }
  return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * 6 * 4096) == cudaSuccess ? 6 * 4096 : -1;
#else
  (void)host;
  (void)n;
  return 0;
#endif
}

int conv_gemm_stages(int npad, int prec) {
  return is_direct(prec) ? stages_prec<kPrecF16Direct>(npad)
         : prec == kPrecF16     ? stages_prec<kPrecF16>(npad)
                                : stages_prec<kPrecTF32>(npad);
}

int conv_gemm_smem_bytes(int npad, int KB, int S, int prec, int n_tiles) {
  const int stages = conv_gemm_stages(npad, prec);
  const int stage_bytes = (is_direct(prec) ? 0 : kABytes) + 2 * npad * (is_f16(prec) ? 64 : 128);
  return 1024 + stages * stage_bytes + tail_bytes(stages, KB, S, n_tiles * npad, npad, is_direct(prec));
}

void launch_conv_gemm(const ConvGemmArgs& a, cudaStream_t st) {
  if (a.prec == kPrecF16Direct && a.src_presplit) launch_prec<kPrecF16Presplit>(a, st);
  else if (a.prec == kPrecF16Direct) launch_prec<kPrecF16Direct>(a, st);
  else if (a.prec == kPrecF16) launch_prec<kPrecF16>(a, st);
  else launch_prec<kPrecTF32>(a, st);
}

}  // namespace cbg
