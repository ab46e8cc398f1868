// common.hpp — shared host/device definitions of the streamconv B200 engine.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/streamconv_b200.h"

namespace scb {

// Typed error carrying an sc_status (1 + streamconv::ErrCode ordinal, error.hpp:8-29).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Exact rational for rate ratios (reference Rational, rational.hpp:13-71: normalized, den>0).
struct Rate {
  int64_t num = 1, den = 1;
  static int64_t gcd(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    while (b) {
      int64_t t = a % b;
      a = b;
      b = t;
    }
    return a;
  }
  void norm() {
    int64_t g = gcd(num, den);
    if (g > 1) {
      num /= g;
      den /= g;
    }
  }
  bool operator==(const Rate& o) const { return num == o.num && den == o.den; }
  bool operator!=(const Rate& o) const { return !(*this == o); }
};

enum ActKind : int { ACT_ID = SC_ACT_IDENTITY, ACT_TANH = SC_ACT_TANH, ACT_LRELU = SC_ACT_LEAKY_RELU };

// ------------------------------------------------------------------------------------------
// Kernel-side parameter block of the generic cached frame-convolution.
//
// Activation buffers are FRAME-MAJOR per stream: [stream][cache + T][C] fp32 — each frame is
// a contiguous channel vector.  One op computes, for every stream s and output row i < t_out:
//
//   out_row(s,i)[n] = post( bias[n] + sum_{q<taps} sum_{c<cin} W[q][c][n] *
//                            pre(in(s, in_f0 + i*row_step + q*tap_step)[in_off + c]) )
//                     + resid(s, res_f0 + i)[res_off + n]
//
// With n < nout.  For a stride-S conv row_step=S, tap_step=d.  A ConvTranspose1d with
// upsampling r is lowered to its polyphase form (taps over input frames, nout = r*Cout): an
// output row of r*Cout floats is exactly r consecutive output frames, so the polyphase
// interleave is free in this layout.  The GATE epilogue pairs columns (2j, 2j+1) ->
// tanh(a)*sigmoid(b) and writes nout/2 values per row.
struct ConvParams {
  const float* in;       // buffer base (stream 0, frame 0, channel 0)
  int64_t in_sstride;    // floats between streams
  int in_fstride;        // floats per frame (buffer channels)
  int in_off;            // channel offset of the view
  int cin;               // channels read per frame
  int in_f0;             // first window frame (cache - P)
  int row_step;          // input frames per output row (conv stride; 1 for convT)
  int tap_step;          // input frames between taps (dilation)
  int taps;              // taps per output row
  const float* w;        // [taps][cin][nout]
  const float* bias;     // [nout]
  int nout;              // GEMM N (r*Cout for convT, 2*C for gate)
  float* out;            // output buffer base
  int64_t out_sstride;   // floats between streams
  int64_t out_base;      // float offset of output row 0 within a stream (cache*C)
  int out_rstride;       // floats per output row (nout, or nout/2 with gate)
  int t_out;             // output rows per stream
  int streams;
  int pre_act;
  float pre_alpha;
  int post_act;
  float post_alpha;
  int gate;              // 1: gated epilogue
  const float* res;      // residual buffer base (nullptr: none)
  int64_t res_sstride;
  int res_fstride;
  int res_off;
  int res_f0;            // frame of output row 0 in the residual buffer (cache - A)
  int res_act;
  float res_alpha;
};

// Per-buffer descriptor for the batched cache-carry and reset kernels.
struct BufDesc {
  float* base;
  int64_t sstride;  // floats per stream
  int64_t item0;    // prefix of streams*C over the table (carry work items)
  int64_t ritem0;   // prefix of C over the table (reset work items, per stream)
  int C;            // floats per frame
  int cache;        // cache frames
  int t;            // frames written this call (carry shift)
  int pad_;
};

}  // namespace scb
