// program.hpp — a causalized model lowered to frame buffers and fused cached-conv ops.
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace scb {

// One activation buffer: per stream [cache + T][C] fp32, frame-major.  `rate` = frames of this
// buffer per input sample, so a call with F input frames writes T = F*rate frames.
struct BufferSpec {
  int C = 1;
  int64_t cache = 0;  // frames kept across calls (max look-back of all readers)
  int64_t align = 1;  // cache is rounded to a multiple of this (strided readers' super-rows)
  Rate rate;
  std::string name;
};

// One fused cached-convolution launch (see ConvParams in common.hpp for the exact formula).
struct ConvOp {
  bool convt = false;        // polyphase ConvTranspose1d
  int in_buf = 0, in_off = 0, cin = 0;
  int out_buf = 0;
  int64_t look = 0;          // window look-back in input frames (causal pad incl. Eq. 2)
  int taps = 1, row_step = 1, tap_step = 1;
  int nout = 0, out_rstride = 0;
  int cout = 0, K = 1, S = 1, d = 1, r = 1;  // original layer geometry
  int pre_act = ACT_ID;
  float pre_alpha = 0.f;
  int post_act = ACT_ID;
  float post_alpha = 0.f;
  bool gate = false;
  int res_buf = -1, res_off = 0, res_act = ACT_ID;
  int64_t res_delay = 0;
  float res_alpha = 0.f;
  // PQMF fast form (hint verified): 1 = analysis, 2 = synthesis; constants below
  int pqmf = 0;
  int pq_A = 0, pq_B = 0, pq_M = 0;  // analysis: A prototype phases x B = 2M modulation rows
  std::vector<float> pq_S;           // analysis [A][B]; synthesis s(q, phi) [Q][M]
  std::vector<float> pq_C;           // analysis Cm [M][B]; synthesis R [classes][M]
  std::vector<int> pq_idx;           // synthesis class of (q, phi) [Q][M]
  int pq_period = 0;                 // synthesis canonical classes (graph.cpp); 0: irregular
  int pq_mirror = 0;
  std::vector<float> w;      // [taps][cin][nout]  (polyphase / gate-interleaved)
  std::vector<float> bias;   // [nout]
  Rate in_rate;              // frames of the input buffer per input sample
  double macs_per_sample = 0;  // algorithmic MACs per input sample (per stream)
  std::string name;
};

struct Program {
  int in_C = 1;
  std::vector<BufferSpec> bufs;  // bufs[0] = source (ingest target)
  std::vector<ConvOp> ops;
  int sink_buf = 0, sink_off = 0, sink_C = 1, sink_act = ACT_ID;
  float sink_alpha = 0.f;
  Rate sink_rate;
  int64_t ratio = 1;          // SPEC compression_ratio
  int64_t latency_sink = 0;   // D_c at the sink, native rate
  int64_t latency_in = 0;     // latency in input samples
  int64_t state_bytes_spec = 0;  // SPEC.md:259 closed form per stream
  double macs_per_sample = 0;
  std::string describe() const;
};

Program lower_graph(const sc_node* nodes, int n_nodes, const float* W, int64_t n_weights,
                    int in_C);

}  // namespace scb
