// runtime.hpp — Plan (causalized model + device weights) and State (device StreamStates).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <tuple>
#include <memory>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "kernels_pqmf.hpp"
#include "kernels_tc.hpp"
#include "program.hpp"

namespace scb {

enum KernelKind { KERNEL_SIMT = 0, KERNEL_TC = 1, KERNEL_PQMF_ANA = 2, KERNEL_PQMF_SYN = 3, KERNEL_SUM = 4 };

struct DevOp {
  float* w = nullptr;
  float* bias = nullptr;
  int kernel = KERNEL_SIMT;
  // tensor-core path (kernel == KERNEL_TC)
  float* wtc = nullptr;      // [2 (hi, lo)][nout][taps_view][cin_view_pad]
  CUtensorMap map_w{};
  int BN = 0;
  bool bf16 = false;
  bool f16 = false;          // fp32 plan, 3xFP16 split (fp16 hi / lo weight planes)
  int f16_sw = 0;            // ... weights scaled by 2^f16_sw
  int view_S = 1;            // super-row factor of the input view (conv stride, or 1)
  int cin_view = 0, cin_view_pad = 0, taps_view = 0, tap_rows = 1;
  int chain = -1;            // fp32: index of the K = 1 conv chained into this op's launch
  int k_chain = 0;           // its K (weights appended along K of this op's weight map)
  int chain_one = 1;         // the chained GEMM accumulates in one TMEM chunk (SC_CHAIN_ONE)
  // PQMF fast form (kernel == KERNEL_PQMF_*): factor arrays inside the weight blob
  float* pq_S = nullptr;
  float* pq_C = nullptr;
  float* pq_idx = nullptr;
  int pq_classes = 0;
  std::vector<float> pq_k;   // the bank's coefficients for the kernel-parameter bank (PqmfCoef)
};

struct Plan {
  Program prog;
  int precision = SC_PREC_FP32;
  int device = 0;
  float* wmem = nullptr;
  std::vector<DevOp> dops;
  std::vector<uint8_t> buf_bf16;  // bf16 plans: buffers touched only by tensor-core ops hold bf16
  std::string desc;
  int fw(size_t b) const { return buf_bf16[b] ? prog.bufs[b].C / 2 : prog.bufs[b].C; }  // words/frame
  ~Plan();
};

struct GraphEntry {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // the nodes carrying the caller's I/O pointers (re-targeted per call): the ingest / egress
  // kernels, or the PQMF analysis / synthesis when the mono I/O is fused into them
  cudaGraphNode_t ingest_node = nullptr, egress_node = nullptr;
  cudaKernelNodeParams ingest_params{}, egress_params{};
  IngestArgs ia{};
  EgressArgs ea{};
  PqmfParams pin{}, pout{};
  uint64_t last_use = 0;
};

struct TcLaunch {
  CUtensorMap map_a{};
  CUtensorMap map_w{};   // this call's weight map when its N tile differs from the plan's (own_w)
  bool own_w = false;
  CUtensorMap map_out{};
  CUtensorMap map_res{};
  TcParams p{};
};

// One call's launch geometry.  Calls whose buffer length F is a multiple of the compression
// ratio all share one CallPlan; shorter buffers cycle through a period of CallPlans (phase
// state: a layer fires only when its input holds enough new frames).
struct CallPlan {
  int64_t F = 0;
  std::vector<int64_t> T;     // new frames per buffer this call
  std::vector<int64_t> pend;  // per op: input frames pending (not yet consumed) before the call
  std::vector<int64_t> t_out; // per op: output rows this call (0: op skipped)
  int64_t egress_row = 0;     // first sink-buffer row emitted this call
  int64_t egress_T = 0;       // sink frames emitted this call
  std::vector<int64_t> pos;   // per buffer: strip row where this call's cache starts
  std::vector<float*> base;   // per buffer: buf_base + pos * C (this call's frame 0 = cache start)
  BufDesc* d_desc = nullptr;  // carry table (wrapped buffers: cache moved to the strip start)
  int n_desc = 0;
  int64_t carry_items = 0;
  int n_launch = 0;           // kernels one call of this plan launches
  int fuse_in = -1;           // the PQMF analysis op that reads the caller's input (no ingest)
  int fuse_out = -1;          // the PQMF synthesis op that writes the caller's output (no egress)
  std::vector<int> chained;   // per op: the op chained into its launch this call (-1: none)
  std::vector<TcLaunch> tc;
  std::map<std::pair<const float*, float*>, GraphEntry> graphs;
  uint64_t last_use = 0;      // LRU stamp (State::plan_clock)
  int64_t dev_bytes = 0;      // device memory this plan owns (carry table)
};

struct State {
  const Plan* plan = nullptr;
  int streams = 0;
  int64_t max_frames = 0;
  float* mem = nullptr;
  int64_t mem_bytes = 0;
  // red zones (SC_REDZONE=1; compute-sanitizer is unavailable on the GPU pool): guard floats
  // after each stream's strip and between buffers, filled with a byte pattern at creation and
  // after a full reset; redzone_check() counts the guard bytes a kernel overwrote.
  bool capturing = false;                // enqueue() is recording a CUDA graph
  int64_t rz_stream = 0;                 // guard floats at the end of every stream's region
  int64_t rz_gap = 0;                    // guard floats before each buffer and after the last
  std::vector<int64_t> rz_used;          // per buffer: used floats per stream (before the guard)
  void redzone_fill(cudaStream_t s);
  int64_t redzone_check();
  int64_t cache_bytes_per_stream = 0;
  std::vector<float*> buf_base;
  std::vector<int64_t> buf_sstride;
  BufDesc* d_desc = nullptr;  // reset table (all cached buffers)
  int n_desc = 0;
  int64_t reset_items = 0;
  int* d_ids = nullptr;
  bool use_graphs = true;
  cudaStream_t capture_stream = nullptr;
  uint64_t use_clock = 0;
  // stream position (all streams advance in lockstep)
  std::vector<int64_t> N;     // cumulative frames written per buffer
  int64_t E = 0;              // cumulative sink frames emitted
  int64_t D = -1;             // sink lag in sink frames (fixed by the first call after reset)
  std::map<std::vector<int64_t>, std::unique_ptr<CallPlan>> plans;
  // The CallPlan cache is bounded: with buffer lengths that keep changing, new geometries keep
  // appearing; beyond kMaxCallPlans the least recently used plan (carry table, graphs) is freed.
  static constexpr size_t kMaxCallPlans = 32;
  uint64_t plan_clock = 0;
  int64_t plan_bytes = 0;      // device bytes owned by cached CallPlans (in sc_state_device_bytes)
  void evict_lru_plan();
  bool phase_mode = false;     // created for buffers shorter than the compression ratio
  std::vector<int64_t> cache;  // per-buffer cache frames of this state
  // Strips: each buffer holds cache + strip_k x T frames per stream; successive calls slide
  // the cache start by T instead of copying the cache back (carry only on wrap-around).
  int strip_k = 1;
  bool carry_slot = false;     // some buffer has a cache: profile layouts carry a carry slot
  int64_t launched = 0;        // kernels launched by this state (eager, captured or replayed)
  std::vector<int64_t> pos;    // per buffer: strip row of the cache start for the next call
  std::vector<BufDesc> reset_desc;  // host copy of the reset table (bases at strip start)

  int64_t lag_for(int64_t F) const;
  void advance(int64_t F, const CallPlan& cp);

  std::vector<int64_t> next_counts(int64_t F) const;
  CallPlan& call_plan(int64_t F);
  ConvParams conv_params(size_t op, const CallPlan& cp) const;
  PqmfParams pqmf_params(size_t op, const CallPlan& cp) const;
  // pqmf_params plus the caller's I/O when this op carries the fused mono input / output
  PqmfParams pqmf_io_params(size_t op, const CallPlan& cp, const float* in, float* out) const;
  SumParams sum_params(size_t op, const CallPlan& cp) const;
  IngestArgs ingest_args(const float* in, const CallPlan& cp) const;
  EgressArgs egress_args(float* out, const CallPlan& cp) const;
  void check_frames(int64_t frames) const;
  void enqueue(const float* in, float* out, CallPlan& cp, cudaStream_t s, cudaEvent_t* ev);
  void profile(const float* in, float* out, int64_t frames, int steps, float* ms, cudaStream_t s);
  int launches(int64_t frames);
  std::string launch_name(int64_t frames, int i);
  void process(const float* in, float* out, int64_t frames, cudaStream_t s);
  // host-buffer path: H2D / compute / D2H on three streams, double-buffered across calls
  void process_host(const float* h_in, float* h_out, int64_t frames, cudaStream_t s);
  void host_wait(cudaStream_t s);
  void process_host_bf16(const uint16_t* h_in, uint16_t* h_out, int64_t frames, cudaStream_t s);
  void process_host_io(const void* h_in, void* h_out, int64_t frames, cudaStream_t s, bool bf16);
  float* io_in[2] = {nullptr, nullptr};
  float* io_out[2] = {nullptr, nullptr};
  uint16_t* io_in16[2] = {nullptr, nullptr};   // bf16 host I/O staging (sc_process_host_bf16)
  uint16_t* io_out16[2] = {nullptr, nullptr};
  int64_t io_in_floats = 0, io_out_floats = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_entry[2] = {}, ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  int64_t host_calls = 0;
  void reset(const int* ids, int n_ids, cudaStream_t s);
  ~State();
};

std::unique_ptr<Plan> make_plan(const sc_node* nodes, int n_nodes, const float* W, int64_t nW,
                                int in_C, int precision, int device);
std::unique_ptr<Plan> make_plan_dag(const sc_gnode* nodes, int n_nodes, const sc_edge* edges,
                                    int n_edges, const float* W, int64_t nW, int in_C,
                                    int precision, int device);
std::unique_ptr<Plan> make_plan(Program prog, int precision, int device);
std::unique_ptr<State> make_state(const Plan* plan, int streams, int64_t max_frames);

// SPEC baseline_ola (ola.cu) and metrics_bench (metrics.cu).
struct Ola {
  std::unique_ptr<Plan> plan;                        // offline program (original pads)
  std::map<int64_t, std::unique_ptr<State>> states;  // by chunks per stream
  int streams = 0;
  int64_t N = 0, hop = 0, max_frames = 0;
  int overlap = 0;
  float* d_in = nullptr;   // gathered chunks [streams * nc][C][N]
  float* d_out = nullptr;  // chunk outputs [streams * nc][C'][N * sink]
  float* d_w = nullptr;    // window, N * sink
  int64_t in_floats = 0, out_floats = 0;
  ~Ola();
};
std::unique_ptr<Ola> make_ola(const sc_gnode* nodes, int n, const sc_edge* edges, int ne, const float* W,
                              int64_t nW, int in_C, int precision, int device, int64_t chunk, int overlap_pct,
                              int streams, int64_t max_frames);
void ola_process(Ola& o, const float* in, float* out, int64_t T, cudaStream_t s);
const Plan& ola_plan(const Ola& o);
std::vector<double> ola_window(int64_t Nw, int overlap_pct);
void signal_moments(const float* x, const float* y, int n, int64_t T, double* moments, cudaStream_t st);
void spectral_distance(const float* x, const float* y, int n, int64_t T, double* out, cudaStream_t st);
void best_lag(const float* ref, const float* test, int n, int64_t T, int max_lag, int64_t* lags, cudaStream_t st);

// tensor_core conv1d (kernels.cpp:73-104) on a device batch, reference layout in and out.
void conv1d_batched(const float* x, int batch, int M, int64_t L, const float* w, const float* b,
                    int N, int K, int S, int d, float* y, cudaStream_t s);

// PQMF filter bank design (pqmf.cpp).
void pqmf_filters(int bands, int taps, float* analysis, float* synthesis, double* prototype);

}  // namespace scb
