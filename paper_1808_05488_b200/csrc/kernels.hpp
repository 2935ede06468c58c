// kernels.hpp — launch interface of the CBinfer sm_100a kernels (host side).
//
// Device data layout (per node, S = streams of the stream set, all contiguous
// [S][...] with per-stream strides):
//   feature maps / states : NHWC fp32, channel stride Cs = round_up(C, 4), so
//                           a pixel's channel vector is one 16-B aligned run;
//                           padded channels hold 0 forever.
//   network input frame   : CHW fp32 (the reference Tensor3 layout), read only
//                           by the first layer's fused ingest+detect kernel.
//   change maps           : bitmaps [H][nw] uint32, nw = ceil(W/32) words per
//                           row; bit (col & 31) of word (row, col >> 5); bits
//                           past W are 0 (common.cuh).
//   index lists           : int32 pixel ids p = row*W + col, a concatenation
//                           of row-major runs (one per compaction band); the
//                           count is a device int32 per stream, accumulated
//                           with atomics and zeroed by begin_frame. Counts
//                           are [S][cnt_stride] (each stream's counters in their
//                           own cache lines: the atomics of different streams
//                           do not contend).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace cbg {

// Kernel launch with programmatic stream serialization (common.cuh pdl_*):
// the next kernel of a frame is scheduled while this one drains; every kernel
// launched this way starts with griddepcontrol.wait. CBG_PDL=0 turns it off.
bool pdl_enabled();
template <typename... P, typename... A>
inline void launch_k(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// Fused change detection on the network-input frame (CHW) against a
// closed-loop / feed-forward state (NHWC), reference change.cpp:20-43.
struct DetectFrameArgs {
  const float* const* x_slot;  // device slot holding the frame pointer [S][C][H][W]
  float* state;        // [S][H][W][Cs]
  uint32_t* map;       // [S][H][nw] bitmap of the input frame's detected pixels, cleared by begin_frame
  int map_plain;       // W % 32 == 0 (4-pixel kernels): words merged in registers, else bits OR-ed in
  int32_t* det_count;  // detected (pre-dilation) pixels of stream s at [s * cnt_stride], atomic (nullable)
  int cnt_stride;      // ints between consecutive streams' counters (one cache line or more each)
  const uint8_t* boot;       // [S] full-update flags for this frame
  int C, Cs, H, W, S;
  const float* tau;    // device [S] per-stream thresholds of this node (set_thresholds needs no re-capture)
  int closed_loop;
  int state_chw;       // state is [S][C][H][W] (unpadded planes) instead of NHWC
  float* amax;         // [S] running max |value written to the state| (atomicMax)
  const uint8_t* const* x8_slot;  // non-null: 8-bit frames [S][H][W][C] (PNM payload order), x = byte/255
  long long x_sstride;  // fp32 frames: elements between streams' frames (C*H*W, or 0 = one frame for all)
  // 8-bit shadow of the state ([S][H][W][C] bytes, the frames' layout), kept
  // by the 8-bit ingest: every state value it writes is byte/255, so the byte
  // is the state. Written on full updates (always) and at changed pixels
  // (when use_state8); use_state8: compare against it instead of the fp32 state.
  uint8_t* state8;
  int use_state8;
};
void launch_detect_frame(const DetectFrameArgs& a, cudaStream_t st);
bool detect_frame_plain_map(int C, int Cs, int W, int state_chw);

// Change detection on an NHWC input produced by a change-based node. Only the
// producer's update set can differ from the state (exact), so
// the kernel walks the producer's index list. dense != 0 (or boot) walks all pixels.
struct DetectListArgs {
  const float* x;            // [S][H][W][Cs]
  float* state;              // [S][H][W][Cs]
  uint32_t* map;             // [S][H][nw] bitmap, cleared by begin_frame, bits OR-ed in
  int32_t* det_count;        // detected pixels, [s * cnt_stride], atomic (nullable)
  const int32_t* prod_idx;   // [S][H*W]  (nullable when dense)
  const int32_t* prod_count; // [s * cnt_stride]
  const uint32_t* frame;
  const uint8_t* boot;
  const uint8_t* dense;      // device flag (nullable = 0): rescan every pixel
  int Cs, H, W, S;
  const float* tau;          // device [S]
  int closed_loop;
  int cnt_stride;
  // pre-split copy of the state for a 3xFP16 GEMM that reads it (nullable):
  // per 4 channels {hi01, hi23, lo01, lo23} fp16 pairs at the state's byte
  // offsets, split with e = f16_scale_exp(amax_in[s]) exactly as the GEMM would.
  uint32_t* split;
  int32_t* split_e;          // [2][S] exponent of the whole copy, by frame parity
  const float* amax_in;      // [S] the GEMM's operand bound
};
void launch_detect_list(const DetectListArgs& a, cudaStream_t st);

// Window dilation (reference change.cpp:45-67, also CB pooling's map,
// layers.cpp:163) fused with the stream compaction of the output map into the
// index list (reference extract_indexes, change.cpp:77-84). One CTA per band
// of `rows` output rows of one stream, one thread per output word, no block
// barriers: each warp's run of the list (row-major) is placed with one
// atomicAdd on the stream's count.
// Up to 4 input maps are OR-ed first (join nodes, network.cpp:366-373).
// Optionally the map and list of a 2x2 / stride-2 max-pool reading this
// node's output map are derived in the same pass (bands are even-aligned, so
// every pooled row lies inside one band).
struct DilateCompactArgs {
  const uint32_t* in_map[4];  // [S][Hin][nwi] bitmaps
  int n_in;
  uint32_t* out_map;          // [S][Hout][nwo] bitmap (every word written)
  int32_t* idx;               // [S][Hout*Wout]
  int32_t* count;             // list length of stream s at [s * cnt_stride], atomic, zeroed by begin_frame
  int cnt_stride;
  const uint8_t* boot;
  int Hin, Win, Hout, Wout, kh, kw, stride, pad;
  int up;                     // > 1: nearest upsampling map (out (j, i) <- in (j/up, i/up)) instead of a window
  int rows;                   // output rows per band (even): one CTA
  int n_bands;                // bands per stream
  int S;
  int threads;                // per CTA (one per output word of the band, <= 512)
  int smem_bytes;             // fused pool: the band's words
  uint32_t* pool_map;         // fused pool (nullable): [S][Hp][nwp]
  int32_t* pool_idx;          // [S][Hp*Wp]
  int32_t* pool_count;        // [s * cnt_stride]
  int Hp, Wp;
};
void launch_dilate_compact(const DilateCompactArgs& a, cudaStream_t st);
// band geometry: rows per band, bands, threads per CTA, shared memory of a
// fused pool (false: the band does not fit in shared memory)
bool dilate_compact_tiling(int Hin, int Win, int Hout, int Wout, int kh, int stride, int Wp, int* rows, int* bands,
                           int* threads, int* smem_bytes);

// Change-based max pooling at the pool's index list (reference layers.cpp:148-179).
struct PoolArgs {
  const float* x;        // [S][Hin][Win][Cs]
  float* out;            // [S][Hout][Wout][Cs]
  const int32_t* idx;    // [S][Hout*Wout]
  const int32_t* count;  // [s * cnt_stride]
  int Cs, Hin, Win, Hout, Wout, size, stride, S;
  int cnt_stride;
};
void launch_pool(const PoolArgs& a, cudaStream_t st);
// Nearest upsampling at the node's index list (extension; PoolArgs with stride = the factor).
void launch_upsample(const PoolArgs& a, cudaStream_t st);

// Add / Concat joins at the join's index list (reference network.cpp:364-398).
struct JoinArgs {
  const float* in[8];
  int in_cs[8];          // channel stride of each parent
  int in_c[8];           // real channels of each parent
  int n_in;
  int is_add;
  float* out;            // [S][H][W][Cs_out]
  int Cs_out;
  const int32_t* idx;
  const int32_t* count;  // [s * cnt_stride]
  int HW, S;
  int cnt_stride;
  float* amax_out;       // [S] running max |written value|
};
void launch_join(const JoinArgs& a, cudaStream_t st);

// Gather + 3xTF32 tcgen05 GEMM + bias/ReLU scatter (reference im2col + gemm +
// update_output: dense.cpp:44-112, layers.cpp:10-31).
struct ConvGemmArgs {
  // staged A path of a 1x1 layer (prec 1): the A rows come by TMA
  // tile::gather4 over this map of the source [S*Hin*Win][Cs] fp32 (box 32
  // elements x 1 row, 128-B swizzle) instead of the fetch warps' cp.async
  CUtensorMap tmap;
  int use_tma;
  const float* src;        // [S][Hin][Win][Cs] column source (state or producer output)
  int src_presplit;        // src is the detect's pre-split copy (DetectListArgs::split), not fp32
  float* out;              // [S][Hout][Wout][Co4]
  const int32_t* idx;      // [S][Hout*Wout]
  const int32_t* count;    // [s * cnt_stride]
  int cnt_stride;
  const uint8_t* wimg;     // pre-swizzled tf32 hi/lo weight images [n_tiles][KB][2][NPAD][128B]
  const uint32_t* ktab;    // [KB*8][2] per 16-B chunk: (kj | ki<<8 | c0<<16 | invalid<<31, (kj*Win + ki)*Cs + c0)
  const float* bias;       // [n_tiles*NPAD]
  int Cs, Hin, Win, Hout, Wout, Co4;
  int stride, pad;
  int kh, kw;              // kernel extent (rows whose whole window is inside the image skip the bounds checks)
  int KB;                  // K blocks of 32 fp32
  int npad;                // N tile: 16, 32, 64, 128 or 256
  int n_tiles;             // ceil(Co4 / npad)
  int relu;
  float slope;             // relu: 0 = ReLU (std::max(v, 0.f)), > 0 = leaky ReLU v * slope (extension)
  int S;
  int grid;                // persistent CTAs (<= SM count)
  int prec;                // 0: 3xTF32, 1: 3xFP16 with power-of-two scaling (conv_tcgen05.cu)
  int w_exp;               // fp16: weights were scaled by 2^-w_exp on the host
  const float* amax_in;    // [S] bound of |source values| (fp16 operand scale)
  float* amax_out;         // [S] running max |written output| (atomicMax), nullable
};
void launch_conv_gemm(const ConvGemmArgs& a, cudaStream_t st);
int conv_gemm_smem_bytes(int npad, int KB, int S, int prec, int n_tiles);
int conv_gemm_stages(int npad, int prec);

// Bit-exact CUDA-core update for narrow layers (Cout <= 16): the reference's
// sequential non-FMA fp32 sum in im2col row order (conv_exact.cu).
struct ConvExactArgs {
  const float* src;        // column source; element (c, j, i) at c*cstride + (j*Win + i)*pstride
  long long src_sstride;   // per-stream stride of src (elements)
  long long cstride;
  int pstride;
  float* out;              // [S][Hout][Wout][Co4]
  const int32_t* idx;      // [S][Hout*Wout]
  const int32_t* count;    // [s * cnt_stride]
  int cnt_stride;
  const float* w;          // [Cout][Cin*kh*kw] (reference weights layout, tensor.hpp:47)
  const float* bias;       // [Cout]
  int Cin, Cout, Co4, kh, kw, stride, pad;
  int Hin, Win, Hout, Wout;
  int relu;
  float slope;             // as ConvGemmArgs::slope
  int S;
  int sm_count;
  float* amax_out;         // [S] running max |written value|
  unsigned long long one_x2 = 0x3f8000003f800000ull;  // {1.0f, 1.0f}, opaque to ptxas (conv_exact.cu)
};
void launch_conv_exact(const ConvExactArgs& a, cudaStream_t st);
int conv_exact_group(int cout);
bool conv_exact_supported(int kw);
size_t conv_exact_smem_bytes(int cout, int K);

// Device frame-counter advance + per-stream boot flags for this frame.
struct BeginFrameArgs {
  uint32_t* frame;
  uint8_t* boot_now;     // [S] out
  uint8_t* boot_req;     // [S] in, cleared
  const uint8_t* dense;  // device flag: every frame is a full update
  uint8_t* rescan_now;   // [n_nodes] out: dense re-detection after a tau change
  uint8_t* rescan_req;   // [n_nodes] in, cleared
  int32_t* counts;       // per-frame atomic counters [S][cnt_stride] (list lengths, detected pixels):
  int n_counts, cnt_stride, keep;  // entries [s][0, keep) (uploaded by the host) stay, the rest are zeroed
  uint4* clear;          // bitmaps written by OR (sparse detections), zeroed
  long long n_clear;     // 16-B units
  int S, n_nodes;
  // the frame's input pointer into the slot the first detect reads (nullable):
  // a captured graph serves any device input, the pointer set per launch as a
  // kernel-node parameter instead of a host-to-device copy of the slot
  const void* in_ptr;
  const void** in_slot;
};
void launch_begin_frame(const BeginFrameArgs& a, cudaStream_t st);
const void* begin_frame_fn();  // the kernel's function (finds its node in a captured graph)

// Delta output of a node (its changed pixels and their output vectors),
// packed contiguously — the layout of the device staging copy and of the
// pinned host buffer:
//   int32 n[S] (padded to 16 B), then per stream s in order: int32 ids[n_s]
//   (padded to 16 B) and float vals[n_s][Cs]
// so the bytes in use are delta_header_bytes(S) + sum_s delta_stream_bytes(n_s, Cs).
struct DeltaArgs {
  const float* out;      // pack: the node's output [S][HW][Cs]
  const int32_t* idx;    // pack: its index list [S][HW]
  const int32_t* count;  // pack: [s * cnt_stride]
  int cnt_stride;
  uint8_t* dst;          // the staging buffer
  uint8_t* host;         // the host buffer (device address of mapped pinned memory)
  long long copied;      // bytes [0, copied) go to the host by DMA; the kernel writes the rest there
  int Cs, S;
  long long HW;
};
#ifdef __CUDACC__
__host__ __device__
#endif
inline size_t delta_header_bytes(int S) { return (static_cast<size_t>(S) * 4 + 15) / 16 * 16; }
#ifdef __CUDACC__
__host__ __device__
#endif
inline size_t delta_stream_bytes(long long n, int Cs) {
  return (static_cast<size_t>(n) * 4 + 15) / 16 * 16 + static_cast<size_t>(n) * Cs * 4;
}
void launch_pack_delta(const DeltaArgs& a, cudaStream_t st);

// Layout conversions for the synchronising readers and standalone uploads.
void launch_nhwc_to_chw(const float* src, float* dst, int C, int Cs, int HW, cudaStream_t st);
void launch_chw_to_nhwc(const float* src, float* dst, int C, int Cs, int HW, cudaStream_t st);

}  // namespace cbg
