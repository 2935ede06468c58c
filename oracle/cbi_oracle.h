/*
 * cbi_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the reference
 * CBinfer hot path (reference: /root/reference/proj/src/{change,dense,layers,network}.cpp).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this. It is the checker, never the thing measured or shipped. Every function
 * cites the reference file:line it restates; arithmetic order follows the
 * reference exactly (fp32, sequential reductions, no FMA: built with
 * -ffp-contract=off), so outputs are bit-identical to the reference build.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against the unmodified reference compiled by oracle/Makefile (oracle/_ref)
 * and against the reference tests' known-answer vectors (tests/golden/).
 */
#ifndef CBI_ORACLE_H_
#define CBI_ORACLE_H_

#include <stdint.h>

#include "cbg.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* cbo_last_error(void);

/* change.cpp:20-43 */
int cbo_detect_changes(const float* x, float* state, int c, int h, int w, float tau, int mode,
                       uint8_t* map_out);
/* change.cpp:45-61 */
int cbo_dilate_window(const uint8_t* m, int h, int w, int kh, int kw, int stride, int pad,
                      int oh, int ow, uint8_t* out);
/* change.cpp:69-75 (oh/ow derived from the spec as ConvSpec::output_height/width) */
int cbo_propagate_changes(const uint8_t* m, int h, int w, const cbg_conv_spec* s, uint8_t* out,
                          int* oh, int* ow);
/* change.cpp:77-84 */
int cbo_extract_indexes(const uint8_t* m, int h, int w, int32_t* rc, int64_t* n);
/* dense.cpp:44-83 (rc NULL = all output pixels) */
int cbo_im2col(const float* x, int c, int h, int w, const cbg_conv_spec* s, const int32_t* rc,
               int64_t n, float* cols);
/* dense.cpp:85-112 with K = make_kernel_matrix(spec) (tensor.cpp:45-56) */
int cbo_gemm(const cbg_conv_spec* s, const float* cols, int64_t n, float* y);
/* layers.cpp:10-31 */
int cbo_update_output(float* prev, int cout, int oh, int ow, const float* y, const int32_t* rc,
                      int64_t n, const float* bias, int fuse_relu);
/* dense.cpp:8-42 */
int cbo_conv2d_dense(const float* x, int c, int h, int w, const cbg_conv_spec* s, float* y);
/* dense.cpp:125-145 */
int cbo_maxpool_to(const float* x, int c, int h, int w, int size, int stride, int oh, int ow,
                   float* y);
/* tensor.cpp:22-28: derived output dim or the pinned one; -1 on invalid */
int cbo_out_dim(int in_dim, int kernel, int stride, int padding, int pinned);

/* Network restatement: convert_to_cb (network.cpp:416-503) + forward_frame
 * (network.cpp:309-414) + reset (274-290) + set_thresholds (263-272). */
typedef struct cbo_net cbo_net;
int cbo_net_create(const cbg_network_spec* spec, const float* taus, int n_taus,
                   const int* policies, int mode, cbo_net** out);
void cbo_net_destroy(cbo_net* n);
int cbo_net_node_count(const cbo_net* n);
int cbo_net_node_shape(const cbo_net* n, int node, int* kind, int* c, int* h, int* w);
int cbo_net_forward(cbo_net* n, const float* frame);
int cbo_net_reset(cbo_net* n);
int cbo_net_set_thresholds(cbo_net* n, const float* taus, int n_taus);
int cbo_net_read_output(const cbo_net* n, int node, float* y);
int cbo_net_read_state(const cbo_net* n, int node, float* y);
int cbo_net_read_changes(const cbo_net* n, int node, uint8_t* map, int32_t* rc, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif
