// common.cuh — device helpers shared by the CBinfer sm_100a kernels.
// Inline PTX for mbarriers, bulk copies (TMA engine), tcgen05 (UMMA/TMEM) and
// acquire/release global accesses. Written for sm_100a only.
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CBG_DEV __device__ __forceinline__
#ifndef CBG_MBAR_SUSPEND_NS
#define CBG_MBAR_SUSPEND_NS 20000
#endif

namespace cbg {

// ---- programmatic dependent launch -------------------------------------------------
// Kernels of a frame are launched with programmatic stream serialization
// (kernels.hpp launch_k); griddepcontrol.wait blocks until the predecessor has
// completed and its memory is visible (a no-op without the attribute). With
// the implicit trigger (the predecessor's exit) this shortens the kernel-to-
// kernel handoff: 60.6k -> 62.3k frames/s. An early launch_dependents
// (CBG_PDL_TRIGGER=1) lets successor CTAs occupy SMs while they wait, which
// starves the other stream groups' kernels: 36-43k.
CBG_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef CBG_PDL_TRIGGER
#define CBG_PDL_TRIGGER 0
#endif
CBG_DEV void pdl_trigger() {
  if (CBG_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define CBG_PDL_ENTRY \
  do {                \
    pdl_wait();       \
    pdl_trigger();    \
  } while (0)

// ---- change bitmaps --------------------------------------------------------------
// A change map is [H][nw] 32-bit words per stream, nw = ceil(W/32): pixel
// (row, col) is bit (col & 31) of word row*nw + (col >> 5); bits past W are 0.
CBG_DEV int map_words(int W) { return (W + 31) >> 5; }
// OR one pixel's bit into a map (maps written this way are cleared by begin_frame)
CBG_DEV void map_set(uint32_t* m, long long p, int W) {
  const uint32_t pi = static_cast<uint32_t>(p), w = static_cast<uint32_t>(W);  // p < H*W < 2^31
  const uint32_t row = pi / w, col = pi - row * w;
  atomicOr(m + row * static_cast<uint32_t>(map_words(W)) + (col >> 5), 1u << (col & 31));
}
// Warp sum of v, one atomicAdd per warp (nullable dst). Every lane must call it.
CBG_DEV void warp_count(int32_t* dst, int v) {
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && dst != nullptr && v) atomicAdd(dst, v);
}

// ---- running magnitude bounds (fp16 GEMM operand scales) -----------------------
// Warp max of v >= 0, one atomicMax per warp (non-negative floats order as ints).
// Every lane of the warp must call it.
CBG_DEV void warp_amax(float* dst, float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && dst != nullptr && v > 0.0f) atomicMax(reinterpret_cast<int*>(dst), __float_as_int(v));
}

// Streaming reads (data read once per frame: frame bytes, a producer's output
// in its consumer's detect or pool): L2 evict-first, so they do not push the
// GEMMs' gathered rows and weight images out of L2 (CBG_EVICT_FIRST=0: plain)
#ifndef CBG_EVICT_FIRST
#define CBG_EVICT_FIRST 1
#endif
CBG_DEV uint64_t l2_stream_policy() {
  uint64_t p = 0;
#if CBG_EVICT_FIRST
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
CBG_DEV float4 ldg_stream_f4(const float* ptr, uint64_t pol) {
  float4 r;
#if CBG_EVICT_FIRST
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(ptr), "l"(pol));
#else
  (void)pol;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(ptr));
#endif
  return r;
}
CBG_DEV uint32_t ldg_stream_u32(const uint32_t* ptr, uint64_t pol) {
  uint32_t r;
#if CBG_EVICT_FIRST
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
#else
  (void)pol;
  r = __ldg(ptr);
#endif
  return r;
}
CBG_DEV float4 ldg_nc_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ---- shared memory / mbarrier -------------------------------------------------------
CBG_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
CBG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CBG_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
CBG_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
CBG_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// The suspend-time hint lets a waiting warp sleep in try_wait (woken when the
// phase completes) instead of re-issuing the probe: many role warps of the GEMM
// wait most of the time, and their spinning took issue slots from the others.
CBG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity), "n"(CBG_MBAR_SUSPEND_NS)
      : "memory");
}
// 1-D bulk copy global -> shared on the TMA engine, completing on an mbarrier.
CBG_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- cp.async (LDGSTS): 16-B async copy with zero-fill (src_bytes = 0) -----------
// (no "memory" clobber: ordering w.r.t. consumers is carried by the mbarrier /
// wait_group that completes the copy, so the compiler may hoist address math)
CBG_DEV void cp_async16(uint32_t dst_smem, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_smem), "l"(src), "r"(src_bytes));
}
// Shared-memory vector accesses without "memory" clobbers (callers order them
// with warp_sync_mem / barriers), so several can be in flight at once.
CBG_DEV float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
CBG_DEV void sts_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}
CBG_DEV uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
CBG_DEV void warp_sync_mem() { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); }
// Arrive on an mbarrier once all prior cp.async of this thread complete (the
// thread itself does not wait); the barrier's expected count covers it (.noinc).
CBG_DEV void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ---- tcgen05 ------------------------------------------------------------------------
CBG_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
CBG_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
CBG_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
CBG_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Same K=32 block with A (hi and lo) in tensor memory ("ts" form): A_hi at
// TMEM columns [a_hi, a_hi+32), A_lo at [a_lo, a_lo+32), lane = row; each
// k-step of 8 tf32 advances A by 8 columns and B by 32 B (2 in 16-B units).
// The tensor core then reads only B from shared memory.
CBG_DEV void umma_tf32x3_kblock_ts(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                   uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b32 ah, %1;\n\tmov.b32 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, 1;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, 1;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, 1;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, 1;\n\t}" ::"r"(d_tmem),
      "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K=32 block of the 3-term fp16 product with A in TMEM: fp16 pairs packed per
// 32-bit column, so a K=16 MMA spans 8 columns; B (K-major SW64, 64-B rows)
// advances 32 B (2 in 16-B units) per k-step.
CBG_DEV void umma_f16x3_kblock_ts(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b32 ah, %1;\n\tmov.b32 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [al], bh, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bh, %5, 1;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [al], bh, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bl, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bh, %5, 1;\n\t}" ::"r"(d_tmem),
      "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accumulate)
      : "memory");
}
// The same product with the two correction terms in their own accumulator
// (N <= 128): one MMA of width 2N takes A_hi against [B_hi; B_lo] (the weight
// image's hi and lo rows are contiguous), filling [main | corr], and one of
// width N adds A_lo * B_hi into corr. 4 MMA instructions per K-block instead
// of 6 (same tensor time), and the truncating fp32 accumulation of the
// hi*hi main sum no longer absorbs the small terms (the epilogue adds the two
// accumulators once, in fp32).
CBG_DEV void umma_f16x3p_kblock_ts(uint32_t d_tmem, uint32_t d_corr, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                   uint32_t idesc2, uint32_t idesc1, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 ah, al;\n\t.reg .b64 bh;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %7, 0;\n\t"
      "mov.b32 ah, %2;\n\tmov.b32 al, %3;\n\tmov.b64 bh, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bh, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [al], bh, %6, 1;\n\t"
      "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah], bh, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [al], bh, %6, 1;\n\t}" ::"r"(d_tmem),
      "r"(d_corr), "r"(a_hi), "r"(a_lo), "l"(b_hi), "r"(idesc2), "r"(idesc1), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 bit, 8 consecutive columns per thread.
CBG_DEV void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread.
CBG_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 16 lanes x 512 bit: thread t writes lane t/4 (+8) columns 2(t%4)..+1 and 8+2(t%4)..+1
// (registers: [lane, cols 2c..] [lane+8, 2c..] [lane, 8+2c..] [lane+8, 8+2c..]).
CBG_DEV void tmem_st_16x256b_x2(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
CBG_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

CBG_DEV void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread.
CBG_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x 32 bit, 32 consecutive columns per thread.
CBG_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
CBG_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core groups 1024 B apart.
// Bit layout: cute/arch/mma_sm100_desc.hpp (SmemDescriptor): start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48), layout type [61,64) (2 = SW128).
CBG_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= static_cast<uint64_t>(1u) << 46;            // descriptor version (sm100)
  d |= static_cast<uint64_t>(2u) << 61;            // SWIZZLE_128B
  return d;
}

// K-major SWIZZLE_64B: rows of 64 B, 8-row core groups 512 B apart (layout type 4).
CBG_DEV uint64_t umma_desc_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(512u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(4u) << 61;            // SWIZZLE_64B
  return d;
}

// Instruction descriptor for kind::tf32, fp32 accumulate, K-major A and B.
// Bit layout: cute/arch/mma_sm100_desc.hpp (InstrDescriptor).
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                                   // c_format = F32
         | (2u << 7)                                 // a_format = TF32
         | (2u << 10)                                // b_format = TF32
         | (static_cast<uint32_t>(N >> 3) << 17)     // n_dim
         | (static_cast<uint32_t>(M >> 4) << 24);    // m_dim
}

// Instruction descriptor for kind::f16 with fp16 A and B, fp32 accumulate, K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4)                                   // c_format = F32
         | (0u << 7)                                 // a_format = F16
         | (0u << 10)                                // b_format = F16
         | (static_cast<uint32_t>(N >> 3) << 17)     // n_dim
         | (static_cast<uint32_t>(M >> 4) << 24);    // m_dim
}

// ---- 3xFP16 operand split (shared by the GEMM and the detect kernels that
// keep a pre-split copy of a GEMM's input state) ---------------------------------
CBG_DEV unsigned long long pack_f32x2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
// Two fp32 values -> packed fp16 hi and lo parts of (x * 2^-e), packed fp32x2
// arithmetic: x*s exact (power of two), hi = fp16_rn, lo = fp16_rn(x*s - hi)
// (ptxas may fuse the multiply into the subtraction: x*s is exact, so the
// result is the same).
CBG_DEV void f16_split2(float x0, float x1, unsigned long long s2, uint32_t& hi, uint32_t& lo) {
  unsigned long long p;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(pack_f32x2(x0, x1)), "l"(s2));
  float p0, p1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(p0), "=f"(p1) : "l"(p));
  const __half2 hh = __floats2half2_rn(p0, p1);
  const float2 hf = __half22float2(hh);
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(p), "l"(pack_f32x2(hf.x, hf.y)));
  float d0, d1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
  const __half2 ll = __floats2half2_rn(d0, d1);
  hi = *reinterpret_cast<const uint32_t*>(&hh);
  lo = *reinterpret_cast<const uint32_t*>(&ll);
}

// Exponent e with bound * 2^-e < 2^15 (fp16 operands stay finite), clamped so
// 2^-e and 2^e are normal floats.
CBG_DEV int f16_scale_exp(float bound) {
  const uint32_t E = (__float_as_uint(bound) >> 23) & 0xFFu;
  if (!(bound > 0.0f) || E == 0xFFu) return 0;
  int e = static_cast<int>(E) - 127 - 14;
  return e < -126 ? -126 : e > 126 ? 126 : e;
}
CBG_DEV float exp2i(int e) { return __uint_as_float(static_cast<uint32_t>(e + 127) << 23); }

}  // namespace cbg
