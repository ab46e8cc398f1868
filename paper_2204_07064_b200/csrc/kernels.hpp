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

// Generic SIMT cached conv (FFMA, fp32 accumulate): narrow layers and the v0 dense path.
void launch_conv_simt(const ConvParams& p, cudaStream_t st);

// Batched cache carry: for every buffer with cache > 0, frames [T, T+cache) -> [0, cache)
// for every stream.  `items` = sum over buffers of streams*C (precomputed).
void launch_carry(const BufDesc* d_bufs, int nbuf, int streams, int64_t items, cudaStream_t st);
// Weights [N][M][K] -> [K][M][N].
void launch_relayout_w(const float* w, int N, int M, int K, float* o, cudaStream_t st);
// Zero the cache frames of the listed streams in every buffer.
void launch_reset_streams(const BufDesc* d_bufs, int nbuf, const int* d_ids, int n_ids,
                          int64_t items_per_stream, cudaStream_t st);

}  // namespace scb
