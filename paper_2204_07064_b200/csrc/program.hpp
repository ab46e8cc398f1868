// program.hpp — a causalized model lowered to frame buffers and fused cached-conv ops.
#pragma once

#include <memory>
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
  int64_t tail = 0;   // offline (OLA) programs: zero frames readers see after the new frames
  Rate rate;
  std::string name;
};

// One input of a Sum launch (OPK_SUM): rows `cache - delay + t` of buffer `buf`, channels
// [off, off + C), with a pending activation applied on load.
struct SumIn {
  int buf = 0, off = 0, act = ACT_ID;
  float alpha = 0.f;
  int64_t delay = 0;
};

enum OpKind { OPK_CONV = 0, OPK_SUM = 1 };

// One fused cached-convolution launch (see ConvParams in common.hpp for the exact formula), or
// one SPEC Sum that no conv epilogue could absorb (kind OPK_SUM: out = post(sum_i in_i)).
struct ConvOp {
  int kind = OPK_CONV;
  std::vector<SumIn> sum_in;  // OPK_SUM operands in port order
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
  int phases = 1;            // output frames per GEMM row: 2 for a densified stride-1 conv
                             // (2-frame super-rows in, 2 output phases out: N doubles)
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
  int64_t sink_delay = 0;     // a Delay in front of the Sink: egress reads rows cache - delay + t
  float sink_alpha = 0.f;
  Rate sink_rate;
  bool offline = false;       // original (non-causal) pads, no causalize delays: the per-chunk
                              // offline_run of the OLA baseline (every call starts from zeros)
  int64_t ratio = 1;          // SPEC compression_ratio
  int64_t latency_sink = 0;   // D_c at the sink, native rate
  int64_t latency_in = 0;     // latency in input samples
  int64_t state_bytes_spec = 0;  // SPEC.md:259 closed form per stream
  double macs_per_sample = 0;
  std::string describe() const;
};

Program lower_graph(const sc_node* nodes, int n_nodes, const float* W, int64_t n_weights,
                    int in_C);

// SPEC graph_ir DAG (include/streamconv_b200.h sc_gnode / sc_edge): analyses and lowering.
struct DagInfo {
  std::vector<int> order;           // topological node order
  std::vector<int> edge_C;          // channels per edge
  std::vector<Rate> edge_rate;      // RateMap per edge
  std::vector<std::vector<int>> in_edge;    // [node][port] -> edge
  std::vector<std::vector<int>> out_edges;  // [node] -> edges, in edge order
  int source = -1, sink = -1;
  int out_C = 0;
  int64_t ratio = 1;
};
DagInfo dag_validate(const sc_gnode* nodes, int n_nodes, const sc_edge* edges, int n_edges,
                     int in_C);
void dag_receptive_field(const sc_gnode* nodes, int n_nodes, const sc_edge* edges, int n_edges,
                         int in_C, int64_t* past, int64_t* future);
// causalize rewrite; returns the total latency in input samples
int64_t dag_causalize(const sc_gnode* nodes, int n_nodes, const sc_edge* edges, int n_edges,
                      int in_C, std::vector<sc_gnode>* out_nodes, std::vector<sc_edge>* out_edges);
Program lower_dag(const sc_gnode* nodes, int n_nodes, const sc_edge* edges, int n_edges,
                  const float* W, int64_t n_weights, int in_C, bool offline = false);

// SPEC model_io (model_io.cpp): JSON manifest + f32 blob.
std::unique_ptr<struct ::sc_model> model_load(const char* manifest_path, const char* blob_path);
void model_save(const char* manifest_path, const char* blob_path, const sc_gnode* nodes, int n,
                const sc_edge* edges, int ne, const float* W, int64_t nW, int in_C);

}  // namespace scb

// The C-ABI model handle: a loaded graph and its weights (owned arrays).
struct sc_model {
  std::vector<sc_gnode> nodes;
  std::vector<sc_edge> edges;
  std::vector<float> weights;
  int32_t in_channels = 0;
};
