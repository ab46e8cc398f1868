// kernels.hpp — launch wrappers of the sm_100a kernels (all asynchronous on `st`).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace scb {

// I/O transposes between the reference layout [stream][C][T] and frame-major buffers.
struct IngestArgs {
  const float* in;   // [streams][C][T]
  float* buf;        // buffer base
  int64_t sstride;   // 4-byte words per stream in the buffer
  int C, T, cache, streams;
  int bf;            // 1: the buffer holds bf16 (bf16 plans)
};
struct EgressArgs {
  const float* buf;
  int64_t sstride;
  int fstride, off, C, T, cache, streams;
  int act;
  float alpha;
  float* out;        // [streams][C][T]
  int bf;            // 1: the buffer holds bf16 (bf16 plans)
};

void launch_ingest(const IngestArgs& a, cudaStream_t st);
void launch_egress(const EgressArgs& a, cudaStream_t st);
const void* ingest_kernel_ptr();
const void* egress_kernel_ptr();
bool is_egress_wide_kernel(const void* f);
bool is_ingest_wide_kernel(const void* f);
bool ingest_wide(const IngestArgs& a);  // launch_ingest picks ingest_wide_kernel
bool egress_wide(const EgressArgs& a);  // launch_egress picks egress_wide_kernel

// Generic SIMT cached conv (FFMA, fp32 accumulate): narrow layers and the v0 dense path.
void launch_conv_simt(const ConvParams& p, cudaStream_t st);

// SPEC Sum that no conv epilogue absorbed: for every stream s, row t < t_out and
// channel c < C:  out(s, t)[c] = post( sum_q act_q(in_q(s, in_f0[q] + t)[in_off[q] + c]) ),
// operands added left to right in port order (fp32), frame-major buffers as in ConvParams.
constexpr int kMaxSumIn = 8;
struct SumParams {
  int n_in;
  const float* in[kMaxSumIn];
  int64_t in_sstride[kMaxSumIn];
  int in_fstride[kMaxSumIn];
  int in_off[kMaxSumIn];
  int in_f0[kMaxSumIn];     // row of output row 0 (cache - delay)
  int act[kMaxSumIn];
  float alpha[kMaxSumIn];
  float* out;
  int64_t out_sstride;
  int64_t out_base;         // cache * C
  int C, t_out, streams;
  int post_act;
  float post_alpha;
};
void launch_sum(const SumParams& p, cudaStream_t st);

// bf16 <-> fp32 element casts for the bf16 host I/O path (to_f32: bf16 -> fp32, else fp32 ->
// bf16 round-to-nearest-even).
void launch_cast(uint16_t* bf, float* f, int64_t n, bool to_f32, cudaStream_t st);

// Batched cache carry: for every buffer with cache > 0, frames [T, T+cache) -> [0, cache)
// for every stream.  `items` = sum over buffers of streams*C (precomputed).
void launch_carry(const BufDesc* d_bufs, int nbuf, int streams, int64_t items, cudaStream_t st);
// Weights [N][M][K] -> [K][M][N].
void launch_relayout_w(const float* w, int N, int M, int K, float* o, cudaStream_t st);
// Zero the cache frames of the listed streams in every buffer.
void launch_reset_streams(const BufDesc* d_bufs, int nbuf, const int* d_ids, int n_ids,
                          int64_t items_per_stream, cudaStream_t st);

}  // namespace scb
