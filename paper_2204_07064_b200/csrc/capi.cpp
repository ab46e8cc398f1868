// capi.cpp — the extern "C" boundary (include/streamconv_b200.h).  No exception crosses it:
// every entry point maps scb::Error to its sc_status and records the message for
// sc_last_error(), formatted like streamconv::Error::what() (error.hpp:59-60).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "kernels_tc.hpp"
#include "runtime.hpp"

struct sc_plan {
  std::unique_ptr<scb::Plan> p;
};
struct sc_state {
  std::unique_ptr<scb::State> s;
};
struct sc_ola {
  std::unique_ptr<scb::Ola> o;
};

namespace {

thread_local std::string g_err;

const char* kNames[] = {"InvalidArgument",       "InputTooShort",
                        "ChannelMismatch",       "CycleDetected",
                        "DanglingNode",          "RateMismatchAtSum",
                        "MalformedGraph",        "NotCausal",
                        "PaddingNotStreamable",  "InternalNonIntegerDelay",
                        "BufferNotMultipleOfRatio", "LengthNotMultipleOfRatio",
                        "ChunkTooSmall",         "LengthMismatch",
                        "ZeroEnergy",            "VersionMismatch",
                        "CorruptBlob",           "SchemaError",
                        "UnsupportedFormat",     "MalformedHeader"};

template <class F>
int guard(F&& f) {
  try {
    f();
    return SC_OK;
  } catch (const scb::Error& e) {
    g_err = std::string(sc_status_name(e.code)) + ": " + e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = std::string("InvalidArgument: ") + e.what();
    return SC_ERR_INVALID_ARGUMENT;
  }
}

void need(bool ok, const char* what) {
  if (!ok) scb::fail(SC_ERR_INVALID_ARGUMENT, what);
}

}  // namespace

extern "C" {

const char* sc_last_error(void) { return g_err.c_str(); }
const char* sc_version(void) { return "streamconv-b200 0.1 (sm_100a)"; }

const char* sc_status_name(int status) {
  if (status == SC_OK) return "OK";
  if (status >= 1 && status <= 20) return kNames[status - 1];
  if (status >= SC_ERR_CUDA_BASE) return "CudaError";
  return "UnknownError";
}

int64_t sc_delay_for_stride(int64_t S, int64_t R, int64_t Dc) {
  if (S < 1 || R < 0 || Dc < 0) return -1;
  return (S - ((R + Dc) % S)) % S;  // Eq. (2)
}

int sc_branch_alignment(const int64_t* D, int32_t n, int64_t* out) {
  return guard([&] {
    need(n >= 1 && D && out, "branch_alignment: empty input");
    int64_t mx = D[0];
    for (int i = 0; i < n; ++i) {
      need(D[i] >= 0, "branch_alignment: negative delay");
      mx = std::max(mx, D[i]);
    }
    for (int i = 0; i < n; ++i) out[i] = mx - D[i];
  });
}

int sc_plan_create(const sc_node* nodes, int32_t n_nodes, const float* weights_host,
                   int64_t n_weights, int32_t in_channels, int32_t precision, int32_t device,
                   sc_plan** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    *out = nullptr;
    auto p = scb::make_plan(nodes, n_nodes, weights_host, n_weights, in_channels, precision, device);
    *out = new sc_plan{std::move(p)};
  });
}

int sc_plan_create_graph(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                         int32_t n_edges, const float* weights_host, int64_t n_weights,
                         int32_t in_channels, int32_t precision, int32_t device, sc_plan** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    *out = nullptr;
    auto p = scb::make_plan_dag(nodes, n_nodes, edges, n_edges, weights_host, n_weights, in_channels,
                                precision, device);
    *out = new sc_plan{std::move(p)};
  });
}

int sc_graph_validate(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                      int32_t in_channels, int64_t* edge_rates, int32_t* out_channels) {
  return guard([&] {
    const scb::DagInfo g = scb::dag_validate(nodes, n_nodes, edges, n_edges, in_channels);
    if (edge_rates)
      for (int e = 0; e < n_edges; ++e) {
        edge_rates[2 * e] = g.edge_rate[e].num;
        edge_rates[2 * e + 1] = g.edge_rate[e].den;
      }
    if (out_channels) *out_channels = g.out_C;
  });
}

int sc_graph_compression_ratio(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                               int32_t n_edges, int32_t in_channels, int64_t* ratio) {
  return guard([&] {
    need(ratio != nullptr, "ratio is null");
    *ratio = scb::dag_validate(nodes, n_nodes, edges, n_edges, in_channels).ratio;
  });
}

int sc_graph_receptive_field(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges,
                             int32_t n_edges, int32_t in_channels, int64_t* past, int64_t* future) {
  return guard([&] {
    need(past && future, "null argument");
    scb::dag_receptive_field(nodes, n_nodes, edges, n_edges, in_channels, past, future);
  });
}

int sc_graph_causalize(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                       int32_t in_channels, sc_gnode* out_nodes, int32_t node_cap, int32_t* n_out_nodes,
                       sc_edge* out_edges, int32_t edge_cap, int32_t* n_out_edges, int64_t* latency) {
  return guard([&] {
    std::vector<sc_gnode> on;
    std::vector<sc_edge> oe;
    const int64_t lat = scb::dag_causalize(nodes, n_nodes, edges, n_edges, in_channels, &on, &oe);
    if (latency) *latency = lat;
    if (n_out_nodes) *n_out_nodes = static_cast<int32_t>(on.size());
    if (n_out_edges) *n_out_edges = static_cast<int32_t>(oe.size());
    if (out_nodes || out_edges) {
      need(out_nodes && out_edges && static_cast<size_t>(node_cap) >= on.size() &&
               static_cast<size_t>(edge_cap) >= oe.size(),
           "causalize: output arrays too small");
      std::copy(on.begin(), on.end(), out_nodes);
      std::copy(oe.begin(), oe.end(), out_edges);
    }
  });
}

int sc_graph_mac_count(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                       int32_t in_channels, int64_t input_samples, int64_t* macs) {
  return guard([&] {
    need(macs != nullptr && input_samples >= 0, "mac_count: bad argument");
    const scb::DagInfo g = scb::dag_validate(nodes, n_nodes, edges, n_edges, in_channels);
    int64_t total = 0;
    for (int e = 0; e < n_edges; ++e) {
      const sc_gnode& nd = nodes[edges[e].to];
      if (nd.kind != SC_G_CONV) continue;
      // the conv's output edge rate = its input edge rate / S
      const scb::Rate r = g.edge_rate[e];
      const int64_t out_len = input_samples * r.num / (r.den * nd.stride);
      total += out_len * nd.out_channels * nd.in_channels * nd.taps;
    }
    *macs = total;
  });
}

int sc_graph_latency(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                     int32_t in_channels, int64_t* samples) {
  return guard([&] {
    need(samples != nullptr, "samples is null");
    int64_t past = 0, future = 0;
    scb::dag_receptive_field(nodes, n_nodes, edges, n_edges, in_channels, &past, &future);
    if (future > 0)
      scb::fail(SC_ERR_NOT_CAUSAL, "the graph sees " + std::to_string(future) +
                                       " future input samples: causalize it first (SPEC.md:218-226)");
    *samples = scb::dag_causalize(nodes, n_nodes, edges, n_edges, in_channels, nullptr, nullptr);
  });
}

int sc_model_load(const char* manifest_path, const char* blob_path, sc_model** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    *out = nullptr;
    *out = scb::model_load(manifest_path, blob_path).release();
  });
}

int sc_model_graph(const sc_model* m, const sc_gnode** nodes, int32_t* n_nodes, const sc_edge** edges,
                   int32_t* n_edges, const float** weights, int64_t* n_weights, int32_t* in_channels) {
  return guard([&] {
    need(m != nullptr, "model is null");
    if (nodes) *nodes = m->nodes.data();
    if (n_nodes) *n_nodes = static_cast<int32_t>(m->nodes.size());
    if (edges) *edges = m->edges.data();
    if (n_edges) *n_edges = static_cast<int32_t>(m->edges.size());
    if (weights) *weights = m->weights.data();
    if (n_weights) *n_weights = static_cast<int64_t>(m->weights.size());
    if (in_channels) *in_channels = m->in_channels;
  });
}

int sc_model_destroy(sc_model* m) {
  return guard([&] { delete m; });
}

int sc_model_save(const char* manifest_path, const char* blob_path, const sc_gnode* nodes, int32_t n_nodes,
                  const sc_edge* edges, int32_t n_edges, const float* weights, int64_t n_weights,
                  int32_t in_channels) {
  return guard([&] {
    scb::model_save(manifest_path, blob_path, nodes, n_nodes, edges, n_edges, weights, n_weights, in_channels);
  });
}

int sc_ola_create(const sc_gnode* nodes, int32_t n_nodes, const sc_edge* edges, int32_t n_edges,
                  const float* weights_host, int64_t n_weights, int32_t in_channels, int32_t precision,
                  int32_t device, int64_t chunk, int32_t overlap_pct, int32_t n_streams, int64_t max_frames,
                  sc_ola** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    *out = nullptr;
    auto o = scb::make_ola(nodes, n_nodes, edges, n_edges, weights_host, n_weights, in_channels, precision, device,
                           chunk, overlap_pct, n_streams, max_frames);
    *out = new sc_ola{std::move(o)};
  });
}

int sc_ola_process(sc_ola* ola, const float* d_in, float* d_out, int64_t frames, void* stream) {
  return guard([&] {
    need(ola && d_in && d_out, "null argument");
    scb::ola_process(*ola->o, d_in, d_out, frames, static_cast<cudaStream_t>(stream));
  });
}

int sc_ola_destroy(sc_ola* ola) {
  return guard([&] { delete ola; });
}

const char* sc_ola_describe(const sc_ola* ola) { return ola ? scb::ola_plan(*ola->o).desc.c_str() : ""; }

int sc_ola_window(int64_t n, int32_t overlap_pct, float* w) {
  return guard([&] {
    need(n >= 1 && w, "window length must be >= 1");
    need(overlap_pct == 0 || overlap_pct == 25 || overlap_pct == 50, "overlap must be 0, 25 or 50");
    const std::vector<double> v = scb::ola_window(n, overlap_pct);
    for (int64_t i = 0; i < n; ++i) w[i] = static_cast<float>(v[i]);
  });
}

double sc_ola_redundancy(int32_t overlap_pct) { return 100.0 / (100.0 - overlap_pct); }

int sc_fidelity(const float* d_ref, const float* d_test, int32_t n, int64_t T, double* l_s, double* l_w,
                double* l_c, void* stream) {
  return guard([&] {
    need(d_ref && d_test && n >= 1 && T >= 1, "fidelity: empty input");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (l_s) scb::spectral_distance(d_ref, d_test, n, T, l_s, st);
    if (l_w || l_c) {
      std::vector<double> m(static_cast<size_t>(n) * 4);
      scb::signal_moments(d_ref, d_test, n, T, m.data(), st);
      bool zero = false;
      for (int i = 0; i < n; ++i) {
        if (l_w) l_w[i] = std::sqrt(m[4 * i]);
        if (l_c) {
          const bool z = m[4 * i + 2] <= 0 || m[4 * i + 3] <= 0;
          zero = zero || z;
          l_c[i] = z ? std::nan("") : m[4 * i + 1] / std::sqrt(m[4 * i + 2] * m[4 * i + 3]);
        }
      }
      if (zero) scb::fail(SC_ERR_ZERO_ENERGY, "correlation of a signal with zero energy");
    }
  });
}

int sc_best_lag(const float* d_ref, const float* d_test, int32_t n, int64_t T, int32_t max_lag, int64_t* lags,
                void* stream) {
  return guard([&] {
    need(d_ref && d_test && lags && n >= 1, "best_lag: null argument");
    scb::best_lag(d_ref, d_test, n, T, max_lag, lags, static_cast<cudaStream_t>(stream));
  });
}

int sc_plan_destroy(sc_plan* plan) {
  return guard([&] { delete plan; });
}

int sc_plan_ratio(const sc_plan* plan, int64_t* ratio) {
  return guard([&] {
    need(plan && ratio, "null argument");
    *ratio = plan->p->prog.ratio;
  });
}

int sc_plan_sink_rate(const sc_plan* plan, int64_t* num, int64_t* den, int32_t* out_channels) {
  return guard([&] {
    need(plan && num && den && out_channels, "null argument");
    *num = plan->p->prog.sink_rate.num;
    *den = plan->p->prog.sink_rate.den;
    *out_channels = plan->p->prog.sink_C;
  });
}

int sc_plan_latency(const sc_plan* plan, int64_t* samples) {
  return guard([&] {
    need(plan && samples, "null argument");
    *samples = plan->p->prog.latency_in;
  });
}

int sc_plan_state_bytes(const sc_plan* plan, int64_t* bytes) {
  return guard([&] {
    need(plan && bytes, "null argument");
    *bytes = plan->p->prog.state_bytes_spec;
  });
}

int sc_plan_macs_per_sample(const sc_plan* plan, double* macs) {
  return guard([&] {
    need(plan && macs, "null argument");
    *macs = plan->p->prog.macs_per_sample;
  });
}

int sc_plan_num_ops(const sc_plan* plan, int32_t* n) {
  return guard([&] {
    need(plan && n, "null argument");
    *n = static_cast<int32_t>(plan->p->prog.ops.size());
  });
}

int sc_plan_op_macs(const sc_plan* plan, int32_t i, double* macs) {
  return guard([&] {
    need(plan && macs, "null argument");
    need(i >= 0 && i < static_cast<int32_t>(plan->p->prog.ops.size()), "op index out of range");
    *macs = plan->p->prog.ops[i].macs_per_sample;
  });
}

const char* sc_plan_describe(const sc_plan* plan) { return plan ? plan->p->desc.c_str() : ""; }

int sc_state_create(const sc_plan* plan, int32_t n_streams, int64_t max_frames, sc_state** out) {
  return guard([&] {
    need(plan && out, "null argument");
    *out = nullptr;
    auto s = scb::make_state(plan->p.get(), n_streams, max_frames);
    *out = new sc_state{std::move(s)};
  });
}

int sc_state_destroy(sc_state* state) {
  return guard([&] { delete state; });
}

int sc_state_reset(sc_state* state, const int32_t* ids, int32_t n_ids, void* stream) {
  return guard([&] {
    need(state != nullptr, "null state");
    state->s->reset(ids, n_ids, static_cast<cudaStream_t>(stream));
  });
}

int sc_state_device_bytes(const sc_state* state, int64_t* bytes) {
  return guard([&] {
    need(state && bytes, "null argument");
    *bytes = state->s->mem_bytes + state->s->plan_bytes;  // state + cached call plans
  });
}

int sc_state_redzone_check(sc_state* state, int64_t* violations) {
  return guard([&] {
    need(state && violations, "null argument");
    *violations = state->s->redzone_check();
  });
}

int sc_state_cache_bytes(const sc_state* state, int64_t* bytes) {
  return guard([&] {
    need(state && bytes, "null argument");
    *bytes = state->s->cache_bytes_per_stream;
  });
}

int sc_process(sc_state* state, const float* d_in, float* d_out, int64_t frames, void* stream) {
  return guard([&] {
    need(state != nullptr, "null state");
    state->s->process(d_in, d_out, frames, static_cast<cudaStream_t>(stream));
  });
}

int sc_process_host(sc_state* state, const float* h_in, float* h_out, int64_t frames, void* stream) {
  return guard([&] {
    need(state != nullptr, "null state");
    state->s->process_host(h_in, h_out, frames, static_cast<cudaStream_t>(stream));
  });
}

int sc_process_host_bf16(sc_state* st, const uint16_t* h_in, uint16_t* h_out, int64_t frames, void* stream) {
  return guard([&] {
    need(st != nullptr, "null state");
    st->s->process_host_bf16(h_in, h_out, frames, static_cast<cudaStream_t>(stream));
  });
}

int sc_process_host_wait(sc_state* state, void* stream) {
  return guard([&] {
    need(state != nullptr, "null state");
    state->s->host_wait(static_cast<cudaStream_t>(stream));
  });
}

int sc_process_launches(const sc_state* state, int64_t frames, int32_t* n) {
  return guard([&] {
    need(state && n, "null argument");
    *n = state->s->launches(frames);
  });
}

int sc_state_launch_total(const sc_state* state, int64_t* total) {
  return guard([&] {
    need(state && total, "null argument");
    *total = state->s->launched;
  });
}

int sc_state_profile(sc_state* state, const float* d_in, float* d_out, int64_t frames, int32_t steps,
                     float* ms_per_launch, void* stream) {
  return guard([&] {
    need(state && ms_per_launch, "null argument");
    state->s->profile(d_in, d_out, frames, steps, ms_per_launch, static_cast<cudaStream_t>(stream));
  });
}

const char* sc_launch_name(const sc_state* state, int64_t frames, int32_t i) {
  // no exception may leave the C ABI: on error the name is "" and sc_last_error() says why
  thread_local std::string name;
  name.clear();
  const int st = guard([&] {
    need(state != nullptr, "null state");
    name = state->s->launch_name(frames, i);
  });
  (void)st;
  return name.c_str();
}

// tests only: the state's device allocation (red-zone checker self-test)
SC_API int sc_debug_state_mem(sc_state* state, void** ptr, int64_t* bytes) {
  return guard([&] {
    need(state && ptr && bytes, "null argument");
    *ptr = state->s->mem;
    *bytes = state->s->mem_bytes;
  });
}

// experiments only: timestamps written by the TC kernel when SC_TC_DEBUG has bit 32
SC_API int sc_debug_tc_trace(long long* host) {
  return guard([&] { scb::tc_trace_dump(host); });
}

int sc_state_set_graphs(sc_state* state, int32_t enabled) {
  return guard([&] {
    need(state != nullptr, "null state");
    state->s->use_graphs = enabled != 0;
  });
}

int sc_conv1d(const float* d_x, int32_t batch, int32_t in_channels, int64_t length, const float* d_w,
              const float* d_b, int32_t out_channels, int32_t taps, int32_t stride, int32_t dilation,
              float* d_y, void* stream) {
  return guard([&] {
    scb::conv1d_batched(d_x, batch, in_channels, length, d_w, d_b, out_channels, taps, stride,
                        dilation, d_y, static_cast<cudaStream_t>(stream));
  });
}

int64_t sc_conv_output_length(int64_t L, int32_t K, int32_t S, int32_t d) {
  // kernels.cpp:46-49
  const int64_t span = static_cast<int64_t>(K - 1) * d + 1;
  return (L - span) / S + 1;
}

int sc_pqmf_filters(int32_t bands, int32_t taps, float* analysis, float* synthesis, double* proto) {
  return guard([&] { scb::pqmf_filters(bands, taps, analysis, synthesis, proto); });
}

}  // extern "C"
