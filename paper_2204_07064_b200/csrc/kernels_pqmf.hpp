// kernels_pqmf.hpp — PQMF analysis / synthesis fast form (kernels_pqmf.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace scb {

struct PqmfParams {
  const float* in;       // input buffer base (stream 0, frame 0)
  int64_t in_sstride;    // floats between streams
  int in_fstride;        // floats per input frame
  int in_off;            // channel offset of the view
  int in_f0;             // first window frame
  const float* S;        // analysis S[A][B]; synthesis s(q, phase) [Q][M]
  const float* C;        // analysis Cm[M][B]; synthesis R[classes][M]
  const float* idx;      // synthesis class index [Q][M] (as float)
  const float* bias;
  int nclass;            // synthesis modulation classes
  int period;            // synthesis canonical class layout (graph.cpp factor_pqmf_synthesis)
  int mirror;
  float* out;
  int64_t out_sstride;
  int64_t out_base;      // float offset of output row 0 within a stream
  int t_out;             // output rows (frames of 16 samples / 16 bands) per stream
  int streams;
  int pre_act;
  float pre_alpha;
  int post_act;
  float post_alpha;
  // fused mono input (analysis, xin != nullptr): window rows >= cache0 (relative to `in`'s
  // frame 0) come from the caller's input xin[stream * xin_T + row - cache0] instead of the
  // state's strip, and rows >= xin_T (the last cache0 rows of the call) are also written to the
  // strip (`strip`, same geometry as `in`): they are the next call's cache.  No ingest launch.
  const float* xin;
  float* strip;
  int xin_T;
  int cache0;
};

// The bank's coefficients, passed by value (kernel-parameter / constant bank):
//   analysis : S[A][B] | Cm[M][B] | bias[M]        (256 + 512 + 16 floats)
//   synthesis: R[classes][M] | s[Q][M] | bias[1]   (<= 512 + 256 + 1 floats)
struct PqmfCoef {
  float c[800];  // with PqmfParams under the classic 4 KB parameter bank (larger params go through LDC)
};

// kind 1 = analysis (A = 8, B = 32), 2 = synthesis (Q = 16, canonical classes, P in {1, 2});
// 16 bands.
bool pqmf_fast_shape(int kind, int bands, int A_or_Q, int B_or_classes, int period = 0, int mirror = 0);
void launch_pqmf(int kind, const PqmfParams& p, const PqmfCoef& k, cudaStream_t st);
// the kernel functions (graph nodes re-targeted per call when they carry the caller's I/O)
const void* pqmf_kernel_ptr(int kind, int period, int mirror);
constexpr int kPqmfLook = 240;  // analysis window look-back (K - M) of the 16-band, 256-tap bank

}  // namespace scb
